#!/bin/bash
# Tile L2 prefetch of columns only / values only vs both; R-MAT with the prefetch forced on (columns only)
mkdir -p gpurun_out; out=gpurun_out/r02_pfwhat.jsonl; : > $out
for i in 1 2; do
  for w in b c v; do ARGCSR_L2PF_WHAT=$w timeout 500 python scripts/bench_configs.py C2 C2:4 C5 >> $out 2>&1; done
  timeout 500 python scripts/bench_configs.py C3 >> $out 2>&1
  for w in c v; do ARGCSR_L2PF=1 ARGCSR_L2PF_WHAT=$w timeout 500 python scripts/bench_configs.py C3 >> $out 2>&1; done
done
