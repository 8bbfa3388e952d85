V="LPD4P1B4 LPD4P0B4 LPD2P0B6 LP4P0B4 U4P0B4"
CONFIGS="C2:1 C2:32 C3:1 C4:1" LAYOUTS="compact" VARIANTS="$V" STEPS=50 timeout 1500 bash scripts/sweep.sh > /dev/null 2>&1
cat gpurun_out/sweep.txt
CONFIGS="C3:1 C4:1" LAYOUTS="compact" VARIANTS="U4P1B4" POLS="x1s1 x1s0 x0s1" STEPS=50 OUT=gpurun_out/sweep_pol.txt timeout 1500 bash scripts/sweep.sh > /dev/null 2>&1
cat gpurun_out/sweep_pol.txt
for w in 0; do ARGCSR_L2_WINDOW=$w python bench.py --config C3 --steps 30 --warmup 5 --no-variants --no-cpu-baseline | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('C3 L2_WINDOW=0', j['ms_per_step'], j['roofline']['frac'])"; done
