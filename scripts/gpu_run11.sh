timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.txt 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
for c in C2 C3 C4 C4f32 C1; do timeout 600 python bench.py --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "$c rc=$?"; done
TAG=r01 CONFIGS="C2:1:compact C2:32:compact C3:1:compact C4:1:compact C1:1:compact C2:1:reference" timeout 1800 bash scripts/profile.sh
