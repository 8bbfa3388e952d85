export PYTHONWARNINGS=ignore
V="U4P0B5 ARGCSR_L2_WINDOW=0 ARGCSR_MAP=0 ARGCSR_XPOL=0 ARGCSR_SPOL=1 U4P0B5"
CONFIGS="C2:1 C2:32" VARIANTS="$V" STEPS=100 timeout 1500 bash scripts/sweep.sh > /dev/null 2>&1
cat gpurun_out/sweep.txt
