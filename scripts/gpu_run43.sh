# r01c evidence: ncu launch lists + --set full per config, summaries built on the box, then the bench lines
export PYTHONWARNINGS=ignore
mkdir -p gpurun_out/prof gpurun_out/bench
TAG=r01c CONFIGS="C2:1:compact C3:1:compact C4:1:compact C4f32:1:compact C1:1:compact C2:32:compact" timeout 2400 bash scripts/profile.sh
python scripts/summarize_profiles.py r01c
cp profiles/r01c_* profiles/ncu_traffic.json gpurun_out/prof/
ls -la gpurun_out
rm -f gpurun_out/r01c_full_C1* gpurun_out/r01c_full_C2* gpurun_out/r01c_full_C3* gpurun_out/r01c_full_C4f32*
for c in C2 C3 C4 C4f32 C1; do timeout 900 python bench.py --config $c > gpurun_out/bench/bench_$c.json 2> gpurun_out/bench/bench_$c.err; echo "$c rc=$?"; done
timeout 900 python bench.py --config C2 --dcs 32 --no-variants > gpurun_out/bench/bench_C2_dcs32.json 2>/dev/null
timeout 1200 python bench.py --config C5 --power-iteration --steps 30 --warmup 3 > gpurun_out/bench/bench_C5.json 2> gpurun_out/bench/bench_C5.err; echo "C5 rc=$?"
timeout 900 python bench.py --impl reference --config C3 --steps 3 --warmup 3 > gpurun_out/bench/bench_reference_C3.json 2>&1
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench/bench_reference_C2.json 2>&1
