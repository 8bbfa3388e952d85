export PYTHONWARNINGS=ignore
V="U4P0B5 ARGCSR_HEAVY_U=8 ARGCSR_HEAVY_U=16"
CONFIGS="C4f32:1" VARIANTS="$V" STEPS=50 timeout 1500 bash scripts/sweep.sh > /dev/null 2>&1
V="U4P0B5 ARGCSR_HEAVY_U=4 ARGCSR_HEAVY_B=5"
CONFIGS="C4:1 C3:1" VARIANTS="$V" STEPS=50 OUT=gpurun_out/sweep2.txt timeout 1500 bash scripts/sweep.sh > /dev/null 2>&1
cat gpurun_out/sweep.txt gpurun_out/sweep2.txt
