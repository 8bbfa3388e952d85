timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.txt 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for c in C2 C3 C4 C4f32 C1; do timeout 900 python bench.py --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "$c rc=$?"; done
timeout 900 python bench.py --config C5 --power-iteration --steps 30 --warmup 3 > gpurun_out/bench_C5.json 2> gpurun_out/bench_C5.err; echo "C5 rc=$?"
timeout 600 python bench.py --impl reference --steps 5 --warmup 2 > gpurun_out/bench_ref_C2.json 2> gpurun_out/bench_ref_C2.err; echo "ref rc=$?"
TAG=r01 CONFIGS="C2:1:compact C2:32:compact C3:1:compact C4:1:compact C1:1:compact" timeout 2400 bash scripts/profile.sh
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/nvsmi.txt
