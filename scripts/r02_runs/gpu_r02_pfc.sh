#!/bin/bash
# Columns-only tile prefetch when x fits (new default) vs both arrays; 256 KB bound on the prefetched bytes (C2 (128,32) now qualifies) vs 128 KB
mkdir -p gpurun_out; out=gpurun_out/r02_pfc.jsonl; : > $out
for i in 1 2; do
  timeout 500 python scripts/bench_configs.py C2 C2:4 C2:32 C1 C4 C4f32 C5 >> $out 2>&1
  ARGCSR_L2PF_WHAT=b timeout 500 python scripts/bench_configs.py C2 C2:4 C2:32 C1 C4 C4f32 >> $out 2>&1
  ARGCSR_L2PF=128 timeout 500 python scripts/bench_configs.py C2:32 >> $out 2>&1
done
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r02_pfc_tests.txt 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/r02_pfc_tests.txt
