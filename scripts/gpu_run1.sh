set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
./scripts/stream_probe > gpurun_out/probe.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.txt 2>&1; echo "tests rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"
CONFIGS="C2:1 C2:32 C3:1 C4:1" VARIANTS="LPD4P1B4 LP4P1B4 U4P1B4 PX4 PX2" STEPS=50 timeout 1200 bash scripts/sweep.sh > /dev/null 2>&1
cat gpurun_out/probe.txt gpurun_out/sweep.txt; tail -3 gpurun_out/gpu_tests.txt
