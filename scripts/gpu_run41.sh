export PYTHONWARNINGS=ignore
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "fp32 or dense_rows or powerlaw or extreme or unit_lengths" 2>&1 | tail -3
V="U4P0B5 ARGCSR_HEAVY_B=5 ARGCSR_HEAVY_U=4"
CONFIGS="C4:1 C4f32:1 C3:1" VARIANTS="$V" STEPS=50 timeout 1500 bash scripts/sweep.sh > /dev/null 2>&1
cat gpurun_out/sweep.txt
