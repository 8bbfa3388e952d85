#!/bin/bash
# Blocked heavy kernel: parity tests of the heavy paths, then C3/C4/C4f32 timings blocked vs lane-walk.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_multigpu_device.py -q -x -p no:cacheprovider -k "heavy or powerlaw or dense or norm2 or fused or one_rank or unit_len" > gpurun_out/r02_heavy_tests.txt 2>&1
echo "tests rc=$?"; tail -5 gpurun_out/r02_heavy_tests.txt
timeout 600 python scripts/bench_configs.py C3 C4 C4f32 C2 > gpurun_out/r02_cfg_blocked.jsonl 2>&1
ARGCSR_HEAVY_BLOCKED=0 timeout 600 python scripts/bench_configs.py C3 C4 C4f32 > gpurun_out/r02_cfg_lanewalk.jsonl 2>&1
cat gpurun_out/r02_cfg_blocked.jsonl gpurun_out/r02_cfg_lanewalk.jsonl
timeout 600 python bench.py --power-iteration --steps 100 --warmup 5 > gpurun_out/r02_bench_C5_pi.json 2> gpurun_out/r02_bench_C5_pi.err
echo "bench rc=$?"; python -c "import json; d=json.loads(open('gpurun_out/r02_bench_C5_pi.json').read().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['power_iteration'])"
