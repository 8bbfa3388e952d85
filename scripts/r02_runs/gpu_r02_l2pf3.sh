#!/bin/bash
# L2 prefetch default rule (x fits the persisting window, tiles <= 256 KB) vs off on every config; full GPU suite
mkdir -p gpurun_out; out=gpurun_out/r02_l2pf3.jsonl; : > $out
for i in 1 2; do
  timeout 400 python scripts/bench_configs.py C2 C2:4 C2:32 C1 C4 C4f32 C3 C5 >> $out 2>&1
  ARGCSR_L2PF=0 timeout 400 python scripts/bench_configs.py C2 C2:4 C2:32 C1 C4 C4f32 C3 C5 >> $out 2>&1
done
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r02_l2pf3_tests.txt 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/r02_l2pf3_tests.txt
cut -c1-110 $out
