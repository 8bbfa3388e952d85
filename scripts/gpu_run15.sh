timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.txt 2>&1; echo "tests rc=$?"
tail -5 gpurun_out/gpu_tests.txt
timeout 900 python bench.py --config C5 --power-iteration --steps 20 --warmup 3 --no-variants --no-cpu-baseline > gpurun_out/bench_C5.json 2> gpurun_out/bench_C5.err; echo "C5 rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/bench_C5.json')); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['format'], d.get('power_iteration'), d['conversion_ms'])"
tail -3 gpurun_out/bench_C5.err
