# fp32 heavy kernel with vector x runs + x remap decision for fp32
export PYTHONWARNINGS=ignore
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "fp32 or dense_rows or unit_lengths or powerlaw" 2>&1 | tail -3
for c in "C4f32 auto" "C4f32 off" "C4f32 on" "C4 auto" "C4 off"; do
  set -- $c
  timeout 300 python bench.py --config $1 --x-remap $2 --steps 50 --warmup 5 --no-variants --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 $2', round(d['ms_per_step'],4), d['value'], d['roofline']['frac'], 'remap', d['format']['x_remap'])"
done
