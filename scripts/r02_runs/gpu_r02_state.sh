#!/bin/bash
# Re-entry check of round 2: full GPU suite, default bench, per-config timings blocked vs lane-walk heavy kernel.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r02_gputests.txt 2>&1
echo "tests rc=$?"; tail -5 gpurun_out/r02_gputests.txt
timeout 600 python scripts/bench_configs.py C3 C4 C4f32 C2 > gpurun_out/r02_cfg_blocked.jsonl 2>&1
ARGCSR_HEAVY_BLOCKED=0 timeout 600 python scripts/bench_configs.py C3 C4 C4f32 > gpurun_out/r02_cfg_lanewalk.jsonl 2>&1
cat gpurun_out/r02_cfg_blocked.jsonl gpurun_out/r02_cfg_lanewalk.jsonl
timeout 900 python bench.py > gpurun_out/r02_bench_default.json 2> gpurun_out/r02_bench_default.err
echo "bench rc=$?"; tail -c 600 gpurun_out/r02_bench_default.json
