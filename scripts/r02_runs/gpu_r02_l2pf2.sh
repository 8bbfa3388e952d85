#!/bin/bash
# L2 prefetch bounded to tiles <= 128 KB and off with unit lengths (the new default) vs off, thresholds 64/256 KB; C1, C2 (dcs 1/4/32), C5
mkdir -p gpurun_out; out=gpurun_out/r02_l2pf2.jsonl; : > $out
for i in 1 2; do
  timeout 300 python scripts/bench_configs.py C2 C2:4 C2:32 C1 C3 >> $out 2>&1
  ARGCSR_L2PF=0 timeout 300 python scripts/bench_configs.py C2 C2:4 C2:32 C1 C3 >> $out 2>&1
done
for t in 64 256; do ARGCSR_L2PF=$t timeout 300 python scripts/bench_configs.py C2 C2:4 >> $out 2>&1; done
timeout 300 python scripts/bench_configs.py C5 >> $out 2>&1
ARGCSR_L2PF=0 timeout 300 python scripts/bench_configs.py C5 >> $out 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_host.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r02_l2pf2_tests.txt 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/r02_l2pf2_tests.txt
cut -c1-120 $out
