#!/bin/bash
# Warp-specialised light kernel: parity with it forced on, then timings.
mkdir -p gpurun_out
ARGCSR_WS=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/r02_ws_tests.txt 2>&1
echo "tests rc=$?"; tail -15 gpurun_out/r02_ws_tests.txt
timeout 300 python scripts/bench_configs.py C2 C2:32 C1 > gpurun_out/r02_ws_cfg.jsonl 2>&1
ARGCSR_WS=0 timeout 300 python scripts/bench_configs.py C2 C2:32 C1 >> gpurun_out/r02_ws_cfg.jsonl 2>&1
ARGCSR_WS=1 timeout 300 python scripts/bench_configs.py C3 C4 >> gpurun_out/r02_ws_cfg.jsonl 2>&1
cat gpurun_out/r02_ws_cfg.jsonl
