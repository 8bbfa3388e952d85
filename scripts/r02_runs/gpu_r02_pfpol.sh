#!/bin/bash
# Tile prefetch with an L2 evict_first hint: R-MAT (forced on, columns / both), C5, C2
mkdir -p gpurun_out; out=gpurun_out/r02_pfpol.jsonl; : > $out
for i in 1 2; do
  timeout 500 python scripts/bench_configs.py C3 C5 C2 >> $out 2>&1
  ARGCSR_L2PF_POL=f timeout 500 python scripts/bench_configs.py C5 C2 >> $out 2>&1
  ARGCSR_L2PF=1 ARGCSR_L2PF_POL=f ARGCSR_L2PF_WHAT=c timeout 500 python scripts/bench_configs.py C3 >> $out 2>&1
  ARGCSR_L2PF=1 ARGCSR_L2PF_POL=f ARGCSR_L2PF_WHAT=b timeout 500 python scripts/bench_configs.py C3 >> $out 2>&1
done
