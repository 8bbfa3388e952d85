#!/bin/bash
# With the tile prefetch: x gathers evict_normal (XPOL=0) and no persisting window, on the configs whose x fits
mkdir -p gpurun_out; out=gpurun_out/r02_xpol2.jsonl; : > $out
for i in 1 2; do
  timeout 500 python scripts/bench_configs.py C2 C2:4 C1 C4 >> $out 2>&1
  ARGCSR_XPOL=0 timeout 500 python scripts/bench_configs.py C2 C2:4 C1 C4 >> $out 2>&1
  ARGCSR_L2_WINDOW=0 ARGCSR_L2PF=1 ARGCSR_L2PF_WHAT=c timeout 500 python scripts/bench_configs.py C2 C2:4 >> $out 2>&1
done
