V="U4P0B5 ARGCSR_MAP=0 ARGCSR_MAP=1"
CONFIGS="C2:1 C2:32 C3:1" LAYOUTS="compact" VARIANTS="$V" STEPS=50 timeout 1500 bash scripts/sweep.sh > /dev/null 2>&1
cat gpurun_out/sweep.txt
