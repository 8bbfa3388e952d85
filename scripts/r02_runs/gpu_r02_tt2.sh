#!/bin/bash
# Light-tile size sweep with the tile L2 prefetch on (512 default, 384, 768, 1024 units)
mkdir -p gpurun_out; out=gpurun_out/r02_tt2.jsonl; : > $out
for i in 1 2; do
  timeout 400 python scripts/bench_configs.py C2 C2:4 C1 >> $out 2>&1
  for t in 384 768 1024; do ARGCSR_TILE_THREADS=$t timeout 400 python scripts/bench_configs.py C2 C2:4 C1 >> $out 2>&1; done
done
