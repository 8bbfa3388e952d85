V="U4P0B4 ARGCSR_HEAVY_U=8"
CONFIGS="C4:1 C3:1" LAYOUTS="compact" VARIANTS="$V" STEPS=40 timeout 1500 bash scripts/sweep.sh > /dev/null 2>&1
cat gpurun_out/sweep.txt
