timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.txt 2>&1; echo "tests rc=$?"
tail -15 gpurun_out/gpu_tests.txt
V="U4P0B4 ARGCSR_BUCKET=0,ARGCSR_SPMV_VARIANT=U4P0B4 U4P1B4 U2P0B6 U4P0B3 ARGCSR_TILE_THREADS=256,ARGCSR_SPMV_VARIANT=U4P0B4 ARGCSR_TILE_THREADS=1024,ARGCSR_SPMV_VARIANT=U4P0B4"
CONFIGS="C3:1 C2:1 C4:1 C2:32" LAYOUTS="compact" VARIANTS="$V" STEPS=50 timeout 1500 bash scripts/sweep.sh > /dev/null 2>&1
cat gpurun_out/sweep.txt
