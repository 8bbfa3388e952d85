export PYTHONWARNINGS=ignore
mkdir -p gpurun_out
for c in "C4f32 auto" "C4f32 on" "C4 auto"; do
  set -- $c
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,launch__registers_per_thread --clock-control none --csv --log-file gpurun_out/l39_$1_$2.csv python bench.py --config $1 --x-remap $2 --steps 2 --warmup 3 --no-variants --no-cpu-baseline > /dev/null 2>&1
done
for e in "ARGCSR_HEAVY_U=16" "ARGCSR_HEAVY_RUNS=0" "ARGCSR_HEAVY_U=8,ARGCSR_HEAVY_RUNS=0"; do
  env ${e//,/ } timeout 300 python bench.py --config C4f32 --steps 50 --warmup 5 --no-variants --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C4f32 $e', round(d['ms_per_step'],4), d['value'])"
done
