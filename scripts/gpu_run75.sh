export PYTHONWARNINGS=ignore
for sp in 0 1 0 1; do for c in C2 C3; do
ARGCSR_ASYNC_SPLIT=$sp timeout 300 python bench.py --config $c --steps 50 --warmup 5 --no-variants --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print('$c split=$sp', e['value'], round(e['ms_per_step'],3))"
done; done
ARGCSR_ASYNC_SPLIT=1 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "host_async" 2>&1 | tail -1
