# TMA-staged heavy kernel: parity + A/B
export PYTHONWARNINGS=ignore
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_multigpu_device.py -m gpu -x -q -k "dense_rows or powerlaw or groups_writes or heavy or unit_lengths" 2>&1 | tail -5
V="U4P0B5 ARGCSR_HEAVY_TMA=1 ARGCSR_HEAVY_TMA=2 ARGCSR_HEAVY_TMA=3"
CONFIGS="C4:1 C4f32:1 C3:1" VARIANTS="$V" STEPS=50 timeout 1500 bash scripts/sweep.sh > /dev/null 2>&1
cat gpurun_out/sweep.txt
