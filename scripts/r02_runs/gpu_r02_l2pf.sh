#!/bin/bash
# Light tiles bulk-prefetch their stored value/column range into L2 (ARGCSR_L2PF=1) vs off, alternating on one box
mkdir -p gpurun_out; out=gpurun_out/r02_l2pf.jsonl; : > $out
for i in 1 2 3; do
  ARGCSR_L2PF=0 timeout 300 python scripts/bench_configs.py C2 C2:32 C4 >> $out 2>&1
  ARGCSR_L2PF=1 timeout 300 python scripts/bench_configs.py C2 C2:32 C4 >> $out 2>&1
done
ARGCSR_L2PF=0 timeout 300 python scripts/bench_configs.py C3 C4f32 >> $out 2>&1
ARGCSR_L2PF=1 timeout 300 python scripts/bench_configs.py C3 C4f32 >> $out 2>&1
ARGCSR_L2PF=1 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r02_l2pf_tests.txt 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/r02_l2pf_tests.txt
cut -c1-130 $out
