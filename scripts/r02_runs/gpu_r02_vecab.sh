#!/bin/bash
# A/B repeat: C3 with V=1 2048-unit tiles vs the default, alternating
mkdir -p gpurun_out; out=gpurun_out/r02_vecab.jsonl; : > $out
for i in 1 2 3; do
  timeout 300 python scripts/bench_configs.py C3 >> $out 2>&1
  ARGCSR_VEC=1 ARGCSR_TILE_THREADS=2048 timeout 300 python scripts/bench_configs.py C3 >> $out 2>&1
  ARGCSR_VEC=1 ARGCSR_TILE_THREADS=1536 timeout 300 python scripts/bench_configs.py C3 >> $out 2>&1
done
cat $out
