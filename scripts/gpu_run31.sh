timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
V="U4P0B5"
CONFIGS="C2:1 C2:32 C3:1 C4:1" LAYOUTS="compact" VARIANTS="$V $V" STEPS=50 timeout 1500 bash scripts/sweep.sh > /dev/null 2>&1
cat gpurun_out/sweep.txt
