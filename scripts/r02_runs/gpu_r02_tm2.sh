#!/bin/bash
mkdir -p gpurun_out; out=gpurun_out/r02_tm2.jsonl; : > $out
timeout 300 python scripts/bench_configs.py C2 C2:32 C4 C4f32 C3 C1 >> $out 2>&1
timeout 300 python scripts/bench_configs.py C2 C3 >> $out 2>&1
cat $out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_multigpu_device.py tests/test_peer.py -q -x -p no:cacheprovider 2>&1 | tail -1
