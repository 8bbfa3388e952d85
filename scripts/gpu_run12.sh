timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.txt 2>&1; echo "tests rc=$?"
tail -15 gpurun_out/gpu_tests.txt
for c in C3 C4 C2; do timeout 600 python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "$c rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/bench_$c.json'))
print('$c', d['value'], 'frac', d['roofline']['frac'], 'fmt', d['format'])
for v in d.get('variants',[]): print('   ', v.get('impl')[:20], v.get('desired_chunk_size'), v.get('layout'), round(v.get('gflops',0),1))
"; done
