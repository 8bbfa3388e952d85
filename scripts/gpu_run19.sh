for c in C4 C4f32; do timeout 600 python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "$c rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/bench_$c.json'))
print('$c', d['value'], 'frac', d['roofline']['frac'], 'remap', d['format']['x_remap'], 'conv', d['conversion_ms'])
for v in d.get('variants',[]): print('   ', v.get('impl')[:20], v.get('desired_chunk_size'), v.get('layout'), v.get('x_remap'), round(v.get('gflops',0),1))
"; done
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,l1tex__throughput.avg.pct_of_peak_sustained_active,launch__registers_per_thread -k regex:spmv_ -s 10 -c 4 --csv python bench.py --config C4f32 --steps 5 --warmup 5 --no-variants --no-cpu-baseline 2>/dev/null | grep -v "^==" | cut -d, -f5,13- | tail -16
