# light tiles with warp-granular dynamic unit chunks (ARGCSR_LIGHT_DYN=1) vs static
export PYTHONWARNINGS=ignore
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "powerlaw" 2>&1 | tail -2
ARGCSR_LIGHT_DYN=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "corpus_grid or stencil or unit_lengths" 2>&1 | tail -2
V="U4P0B5 ARGCSR_LIGHT_DYN=1"
CONFIGS="C3:1 C2:1 C2:32 C4:1" VARIANTS="$V" STEPS=100 timeout 1500 bash scripts/sweep.sh > /dev/null 2>&1
cat gpurun_out/sweep.txt
