#!/bin/bash
# NORM-templated kernels (C2 regression check) + pipelined lane-walk heavy variants.
mkdir -p gpurun_out
timeout 300 python scripts/bench_configs.py C2 C3 C4 C4f32 > gpurun_out/r02_pipe_default.jsonl 2>&1
for p in 8 4 6; do
ARGCSR_HEAVY_PIPE=$p timeout 300 python scripts/bench_configs.py C3 C4 C4f32 > gpurun_out/r02_pipe_$p.jsonl 2>&1
done
cat gpurun_out/r02_pipe_*.jsonl
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_multigpu_device.py tests/test_peer.py -q -x -p no:cacheprovider -k "heavy or norm or fused or scale or power or peer" > gpurun_out/r02_pipe_tests.txt 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/r02_pipe_tests.txt
