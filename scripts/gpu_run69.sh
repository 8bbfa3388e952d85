# e2e through the multi-GPU API (exercised at N=1 via ARGCSR_BENCH_DIST=1) + default bench still intact
export PYTHONWARNINGS=ignore
ARGCSR_BENCH_DIST=1 timeout 600 python bench.py --config C2 --steps 20 --warmup 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('dist N=1', d['ms_per_step'], d['value'], d['e2e'], d['config']['parallelism'])"
timeout 600 python bench.py --steps 50 --warmup 5 --no-variants --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('default', d['ms_per_step'], d['value'], d['e2e']['value'])"
