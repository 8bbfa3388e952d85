# heavy stream at high priority by default: confirm + priority on the light stream too
export PYTHONWARNINGS=ignore
V="U4P0B5 ARGCSR_AUX_PRIO=def"
CONFIGS="C4:1 C4f32:1 C3:1 C2:1 C4:4" VARIANTS="$V" STEPS=100 timeout 1500 bash scripts/sweep.sh > /dev/null 2>&1
cat gpurun_out/sweep.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "powerlaw or dense_rows or fused or host" 2>&1 | tail -2
