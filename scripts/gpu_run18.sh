timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.txt 2>&1; echo "tests rc=$?"
tail -5 gpurun_out/gpu_tests.txt
for c in C4 C4f32 C3 C2; do timeout 600 python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "$c rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/bench_$c.json'))
print('$c', d['value'], 'frac', d['roofline']['frac'], 'remap', d['format']['x_remap'], 'conv', d['conversion_ms'])
for v in d.get('variants',[]): print('   ', v.get('impl')[:20], v.get('desired_chunk_size'), v.get('layout'), v.get('x_remap'), round(v.get('gflops',0),1))
"; done
