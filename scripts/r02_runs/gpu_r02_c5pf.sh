#!/bin/bash
# C5 on one GPU (x = 262 MB): tile L2 prefetch with x gathers at L2 evict_normal / window off
mkdir -p gpurun_out; out=gpurun_out/r02_c5pf.jsonl; : > $out
for i in 1 2; do
  timeout 400 python scripts/bench_configs.py C5 >> $out 2>&1
  ARGCSR_XPOL=0 timeout 400 python scripts/bench_configs.py C5 >> $out 2>&1
  ARGCSR_XPOL=0 ARGCSR_L2PF=1 timeout 400 python scripts/bench_configs.py C5 >> $out 2>&1
  ARGCSR_XPOL=0 ARGCSR_L2_WINDOW=0 ARGCSR_L2PF=1 timeout 400 python scripts/bench_configs.py C5 >> $out 2>&1
  ARGCSR_XPOL=0 ARGCSR_L2_WINDOW=0 ARGCSR_L2PF=1 ARGCSR_SPOL=1 timeout 400 python scripts/bench_configs.py C5 >> $out 2>&1
done
