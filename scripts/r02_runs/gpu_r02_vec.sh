#!/bin/bash
# Unit width V (lanes per thread vector) and tile size: warp x-gather locality vs loads in flight.
mkdir -p gpurun_out; out=gpurun_out/r02_vec.jsonl; : > $out
timeout 300 python scripts/bench_configs.py C2 C4 C3 >> $out 2>&1
for v in 1 2; do for t in 512 1024 2048; do
  ARGCSR_VEC=$v ARGCSR_TILE_THREADS=$t timeout 300 python scripts/bench_configs.py C2 C4 C3 >> $out 2>&1
done; done
cat $out
ARGCSR_VEC=1 ARGCSR_TILE_THREADS=2048 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "stencil27 or powerlaw or corpus_grid or fp32" 2>&1 | tail -1
