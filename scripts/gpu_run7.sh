timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.txt 2>&1; echo "tests rc=$?"
tail -5 gpurun_out/gpu_tests.txt
V="ARGCSR_TMA_CTAS=2 ARGCSR_TMA_CTAS=3,ARGCSR_TMA_STAGE=24000 ARGCSR_TMA_CTAS=2,ARGCSR_TMA_STAGE=48000 ARGCSR_TMA_CTAS=1,ARGCSR_TMA_THREADS=512,ARGCSR_TMA_STAGE=56000 LPD4P1B4"
CONFIGS="C2:1 C2:32 C3:1 C4:1" LAYOUTS="compact" VARIANTS="$V" STEPS=50 timeout 1500 bash scripts/sweep.sh > /dev/null 2>&1
cat gpurun_out/sweep.txt
ncu --set full --clock-control none --import-source on -k regex:spmv_tma -s 6 -c 1 -o gpurun_out/tma_C2c python bench.py --config C2 --steps 5 --warmup 3 --no-variants --no-cpu-baseline > /dev/null 2>&1
