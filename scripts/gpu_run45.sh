# paired short-chunk units (one batch for a thread's two units when every chunk of the tile <= U/2)
export PYTHONWARNINGS=ignore
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_multigpu_device.py tests/test_peer.py -m gpu -x -q 2>&1 | tail -3
V="U4P0B5 ARGCSR_PAIR=0"
CONFIGS="C1:1 C4:1 C4f32:1 C2:1 C3:1 C2:32" VARIANTS="$V" STEPS=100 timeout 1500 bash scripts/sweep.sh > /dev/null 2>&1
cat gpurun_out/sweep.txt
