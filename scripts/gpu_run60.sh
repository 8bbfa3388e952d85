# final bench lines (heavy stream priority default) + launch lists for C4/C4f32
export PYTHONWARNINGS=ignore
mkdir -p gpurun_out/bench gpurun_out/prof
for c in C4 C4f32 C3; do timeout 900 python bench.py --config $c > gpurun_out/bench/bench_$c.json 2> gpurun_out/bench/bench_$c.err; echo "$c rc=$?"; done
timeout 900 python bench.py --config C4 --dcs 4 --no-variants > gpurun_out/bench/bench_C4_dcs4.json 2>/dev/null
for c in C4 C4f32; do
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/r01f_launches_${c}_dcs1_compact.csv python bench.py --config $c --steps 5 --warmup 3 --no-variants --no-cpu-baseline > /dev/null 2>&1
done
timeout 600 python bench.py > gpurun_out/bench/bench_default.json 2>/dev/null
