# r01d final evidence: ncu (launch lists + --set full) for the kernels changed since r01c, then all bench lines
export PYTHONWARNINGS=ignore
mkdir -p gpurun_out/prof gpurun_out/bench
TAG=r01d CONFIGS="C1:1:compact C4:1:compact C3:1:compact C2:1:compact" timeout 2400 bash scripts/profile.sh
python scripts/summarize_profiles.py r01d
cp profiles/r01d_* profiles/ncu_traffic.json gpurun_out/prof/
rm -f gpurun_out/r01d_full_*
for c in C2 C3 C4 C4f32 C1; do timeout 900 python bench.py --config $c > gpurun_out/bench/bench_$c.json 2> gpurun_out/bench/bench_$c.err; echo "$c rc=$?"; done
timeout 900 python bench.py --config C2 --dcs 32 --no-variants > gpurun_out/bench/bench_C2_dcs32.json 2>/dev/null
timeout 900 python bench.py --config C4 --dcs 4 --no-variants > gpurun_out/bench/bench_C4_dcs4.json 2>/dev/null
timeout 1200 python bench.py --config C5 --power-iteration --steps 30 --warmup 3 > gpurun_out/bench/bench_C5.json 2> gpurun_out/bench/bench_C5.err
timeout 1200 python bench.py --config C5 --power-iteration --exchange p2p --steps 30 --warmup 3 > gpurun_out/bench/bench_C5_p2p.json 2> gpurun_out/bench/bench_C5_p2p.err
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench/bench_reference_C2.json 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
