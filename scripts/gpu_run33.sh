timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "host_staged" 2>&1 | tail -3
for c in C2 C1 C3; do timeout 600 python bench.py --config $c --steps 50 --no-variants --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', d['value'], d['e2e'])"; done
