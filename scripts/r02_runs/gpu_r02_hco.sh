#!/bin/bash
# Shared-memory carve-out of the long-chunk kernels only (more L1 for the lanes' x lines): 0 / 10 / 25 % vs driver default
mkdir -p gpurun_out; out=gpurun_out/r02_hco.jsonl; : > $out
for i in 1 2; do
  timeout 500 python scripts/bench_configs.py C4f32 C4 C3 >> $out 2>&1
  for c in 0 10 25; do ARGCSR_HEAVY_CARVEOUT=$c timeout 500 python scripts/bench_configs.py C4f32 C4 C3 >> $out 2>&1; done
done
