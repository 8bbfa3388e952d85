# async host SpMV stream: parity + e2e per config
export PYTHONWARNINGS=ignore
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "host_async or host_staged" 2>&1 | tail -2
for c in C2 C3 C4 C1; do
  timeout 300 python bench.py --config $c --steps 50 --warmup 5 --no-variants --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print('$c', round(d['ms_per_step'],4), d['value'], 'e2e', e['value'], round(e['ms_per_step'],3), 'single', e['single_call']['value'])"
done
