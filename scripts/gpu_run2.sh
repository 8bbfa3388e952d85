timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.txt 2>&1; echo "tests rc=$?"
tail -15 gpurun_out/gpu_tests.txt
CONFIGS="C2:1 C2:32 C3:1 C4:1 C1:1" LAYOUTS="compact reference" VARIANTS="LPD4P1B4 U4P1B4" STEPS=50 timeout 1500 bash scripts/sweep.sh > /dev/null 2>&1
cat gpurun_out/sweep.txt
