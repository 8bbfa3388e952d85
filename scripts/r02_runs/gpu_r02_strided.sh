#!/bin/bash
mkdir -p gpurun_out; out=gpurun_out/r02_strided.jsonl; : > $out
timeout 300 python scripts/bench_configs.py C2 C4 C3 C2:32 >> $out 2>&1
ARGCSR_STRIDED=2 timeout 300 python scripts/bench_configs.py C2 C4 C3 C2:32 >> $out 2>&1
cat $out
ARGCSR_STRIDED=2 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "stencil27 or powerlaw or corpus_grid or fp32 or dense_rows or groups_writes" 2>&1 | tail -1
