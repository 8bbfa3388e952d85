# heavy kernel variants at 4 CTAs/SM (U=8) + faster x' gather
export PYTHONWARNINGS=ignore
V="U4P0B5 ARGCSR_HEAVY_U=8,ARGCSR_HEAVY_RUNS=0 ARGCSR_HEAVY_U=16,ARGCSR_HEAVY_RUNS=0 ARGCSR_HEAVY_U=8,ARGCSR_HEAVY_RUNS=1 ARGCSR_HEAVY_U=16,ARGCSR_HEAVY_RUNS=1"
CONFIGS="C4:1 C4f32:1 C3:1 C4:4" VARIANTS="$V" STEPS=50 timeout 1500 bash scripts/sweep.sh > /dev/null 2>&1
cat gpurun_out/sweep.txt
