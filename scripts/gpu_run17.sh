V="U4P0B4 U8P1B2 U8P0B2 U8P0B3 U6P0B3"
CONFIGS="C3:1 C4:1 C2:1" LAYOUTS="compact" VARIANTS="$V" STEPS=40 timeout 1500 bash scripts/sweep.sh > /dev/null 2>&1
cat gpurun_out/sweep.txt
