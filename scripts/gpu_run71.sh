export PYTHONWARNINGS=ignore
mkdir -p gpurun_out/bench
for c in C4 C4f32 C3; do timeout 900 python bench.py --config $c > gpurun_out/bench/bench_$c.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/bench/bench_$c.json')); print('$c', d['ms_per_step'], d['value'], d['roofline']['frac'], d['e2e']['value'], d.get('cpu_baseline',{}).get('parity'))"; done
timeout 900 python bench.py --config C4 --dcs 4 --no-variants > gpurun_out/bench/bench_C4_dcs4.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/bench/bench_C4_dcs4.json')); print('C4dcs4', d['ms_per_step'], d['value'], d['roofline']['frac'])"
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "powerlaw or dense_rows" 2>&1 | tail -1
