#!/bin/bash
mkdir -p gpurun_out; out=gpurun_out/r02_split.jsonl; : > $out
for sp in 0 4 3; do ARGCSR_SPLIT=$sp timeout 300 python scripts/bench_configs.py C2 C2:32 C1 >> $out 2>&1; done
cat $out
ARGCSR_SPLIT=4 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "stencil27 or corpus_grid or fp32 or e8 or empty or zero or extreme or rectangular" 2>&1 | tail -1
