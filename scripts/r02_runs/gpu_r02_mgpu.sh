#!/bin/bash
# GPU checks of the multi-GPU C-ABI layer (run under gpurun from the repo root).
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_multigpu_device.py tests/test_peer.py -q -x -p no:cacheprovider > gpurun_out/r02_mgpu_tests.txt 2>&1
echo "tests rc=$?"
tail -15 gpurun_out/r02_mgpu_tests.txt
timeout 600 python bench.py --power-iteration --steps 100 --warmup 5 > gpurun_out/r02_bench_C5_pi.json 2> gpurun_out/r02_bench_C5_pi.err
echo "bench rc=$?"
tail -c 1500 gpurun_out/r02_bench_C5_pi.err
