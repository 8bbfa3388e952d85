ARGCSR_TILE_THREADS=32 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_multigpu_device.py -m gpu -x -q 2>&1 | tail -3
V="U4P0B5 ARGCSR_TILE_THREADS=32 ARGCSR_TILE_THREADS=64 ARGCSR_TILE_THREADS=32,ARGCSR_WARP_B=6 ARGCSR_TILE_THREADS=32,ARGCSR_WARP_B=4"
CONFIGS="C2:1 C3:1 C4:1 C2:32 C1:1" LAYOUTS="compact" VARIANTS="$V" STEPS=50 timeout 1500 bash scripts/sweep.sh > /dev/null 2>&1
cat gpurun_out/sweep.txt
