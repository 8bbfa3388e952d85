export PYTHONWARNINGS=ignore
V="U4P0B5 ARGCSR_SPOL=0 U4P0B5 ARGCSR_SPOL=0 U4P0B5 ARGCSR_SPOL=0"
CONFIGS="C3:1 C4:1" VARIANTS="$V" STEPS=50 timeout 1500 bash scripts/sweep.sh > /dev/null 2>&1
cat gpurun_out/sweep.txt
