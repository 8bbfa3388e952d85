#!/bin/bash
# Final prefetch rule (columns only on regular matrices with x in the window, both arrays otherwise; tile bound 256 KB of both arrays) vs both arrays
mkdir -p gpurun_out; out=gpurun_out/r02_pfc2.jsonl; : > $out
for i in 1 2; do
  timeout 500 python scripts/bench_configs.py C2 C2:4 C2:32 C4 C1 >> $out 2>&1
  ARGCSR_L2PF_WHAT=b timeout 500 python scripts/bench_configs.py C2 C2:4 C2:32 C4 C1 >> $out 2>&1
done
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "l2_policy or stencil or powerlaw" > gpurun_out/r02_pfc2_tests.txt 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/r02_pfc2_tests.txt
