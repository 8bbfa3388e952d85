#!/bin/bash
mkdir -p gpurun_out; out=gpurun_out/r02_wtile.jsonl; : > $out
for w in 0 5 4 6; do ARGCSR_WTILE=$w timeout 300 python scripts/bench_configs.py C2 C2:32 C4 C4f32 C3 C1 >> $out 2>&1; done
cat $out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_fullsize_parity.py tests/test_multigpu_device.py -q -x -p no:cacheprovider 2>&1 | tail -2
