# heavy/light co-residence: padded heavy shared memory, aux stream priority
export PYTHONWARNINGS=ignore
V="U4P0B5 ARGCSR_HEAVY_SMEM=60000 ARGCSR_HEAVY_SMEM=75000 ARGCSR_HEAVY_SMEM=110000 ARGCSR_AUX_PRIO=hi ARGCSR_AUX_PRIO=lo ARGCSR_AUX_PRIO=hi,ARGCSR_HEAVY_SMEM=60000"
CONFIGS="C4:1 C3:1 C4f32:1" VARIANTS="$V" STEPS=50 timeout 1500 bash scripts/sweep.sh > /dev/null 2>&1
cat gpurun_out/sweep.txt
