timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "heavy or powerlaw or dense or corpus_grid" 2>&1 | tail -2
V="U4P0B5 ARGCSR_HEAVY_K=0 ARGCSR_HEAVY_K=1 ARGCSR_HEAVY_K=2.5 ARGCSR_HEAVY_K=4"
CONFIGS="C3:1 C4:1 C4f32:1" LAYOUTS="compact" VARIANTS="$V" STEPS=50 timeout 1500 bash scripts/sweep.sh > /dev/null 2>&1
cat gpurun_out/sweep.txt
