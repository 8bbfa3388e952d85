export PYTHONWARNINGS=ignore
timeout 900 python -m pytest tests/test_multigpu_device.py tests/test_peer.py -m gpu -x -q 2>&1 | tail -2
mkdir -p gpurun_out/bench
timeout 1200 python bench.py --config C5 --power-iteration --steps 30 --warmup 3 > gpurun_out/bench/bench_C5.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/bench/bench_C5.json')); print(d['ms_per_step'], d['value'], d['roofline']['frac'], d['power_iteration'])"
