#!/bin/bash
# V=4 light kernel at 4 / 6 CTAs per SM vs 5 with the tile prefetch on
mkdir -p gpurun_out; out=gpurun_out/r02_minb.jsonl; : > $out
for i in 1 2; do
  for b in 5 4 6; do ARGCSR_LIGHT_MINB=$b timeout 500 python scripts/bench_configs.py C2 C2:4 C2:32 C5 C4 >> $out 2>&1; done
done
