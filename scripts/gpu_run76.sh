export PYTHONWARNINGS=ignore
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "host_async or host_staged" 2>&1 | tail -1
mkdir -p gpurun_out/bench
timeout 900 python bench.py > gpurun_out/bench/bench_C2.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/bench/bench_C2.json')); print(d['ms_per_step'], d['value'], d['roofline']['frac'], d['e2e']['value'], d['cpu_baseline']['value'], d['cpu_baseline']['parity'])"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
