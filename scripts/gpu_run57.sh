export PYTHONWARNINGS=ignore
for r in auto on; do for c in C3; do
timeout 300 python bench.py --config $c --x-remap $r --steps 50 --warmup 5 --no-variants --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c remap=$r', round(d['ms_per_step'],4), d['value'], d['roofline']['frac'], d['format']['x_remap'], d['format']['x_used_columns'])"
done; done
