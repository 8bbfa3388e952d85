# regression check of the peer epilogue (npeers = 0) on the default path
export PYTHONWARNINGS=ignore
CONFIGS="C2:1 C4:1 C1:1 C3:1" VARIANTS="U4P0B5" STEPS=100 timeout 1500 bash scripts/sweep.sh > /dev/null 2>&1
cat gpurun_out/sweep.txt
for ex in auto p2p; do
timeout 600 python bench.py --config C5 --power-iteration --exchange $ex --steps 20 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C5 $ex N=1', d['ms_per_step'], d['value'], d['roofline']['frac'])"
done
