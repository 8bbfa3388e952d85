#!/bin/bash
mkdir -p gpurun_out; out=gpurun_out/r02_utab.jsonl; : > $out
for u in 0 1 4; do ARGCSR_UTAB=$u timeout 300 python scripts/bench_configs.py C2 C2:32 C4 C3 >> $out 2>&1; done
cat $out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_fullsize_parity.py -q -x -p no:cacheprovider -k "stencil or powerlaw or corpus_grid or fp32 or dense_rows or groups_writes or c2 or c1 or extreme" 2>&1 | tail -1
ARGCSR_UTAB=4 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "stencil27 or corpus_grid or fp32" 2>&1 | tail -1
