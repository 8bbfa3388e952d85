#!/bin/bash
# x beyond the persisting window (C5 on one GPU, R-MAT): window off, tile L2 prefetch on/off, vs the default
mkdir -p gpurun_out; out=gpurun_out/r02_l2pf4.jsonl; : > $out
for i in 1 2; do
  timeout 400 python scripts/bench_configs.py C5 C3 >> $out 2>&1
  ARGCSR_L2_WINDOW=0 timeout 400 python scripts/bench_configs.py C5 C3 >> $out 2>&1
  ARGCSR_L2_WINDOW=0 ARGCSR_L2PF=1 timeout 400 python scripts/bench_configs.py C5 C3 >> $out 2>&1
  ARGCSR_L2_WINDOW=0 ARGCSR_L2PF=64 timeout 400 python scripts/bench_configs.py C5 C3 >> $out 2>&1
done
