#!/bin/bash
mkdir -p gpurun_out; out=gpurun_out/r02_lpipe.jsonl; : > $out
for p in 2 3 4; do ARGCSR_LIGHT_PIPE=$p timeout 300 python scripts/bench_configs.py C3 C2 C4 >> $out 2>&1; done
for p in a b; do ARGCSR_HEAVY_PIPE=$p timeout 300 python scripts/bench_configs.py C4f32 >> $out 2>&1; done
timeout 300 python scripts/bench_configs.py C4f32 >> $out 2>&1
cat $out
for p in 2 4; do ARGCSR_LIGHT_PIPE=$p timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "stencil27 or powerlaw or fp32 or dense_rows or corpus_grid" 2>&1 | tail -1; done
ARGCSR_HEAVY_PIPE=a timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "powerlaw or fp32 or dense_rows" 2>&1 | tail -1
