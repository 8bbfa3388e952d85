#!/bin/bash
# Tile prefetch ahead by ARGCSR_L2PF_AHEAD quarter waves of resident CTAs (0 = own tile, the default) + metadata of that tile
mkdir -p gpurun_out; out=gpurun_out/r02_ahead.jsonl; : > $out
for i in 1 2; do
  for a in 0 1 2 4 8; do ARGCSR_L2PF_AHEAD=$a timeout 500 python scripts/bench_configs.py C2 C2:4 C1 C4 >> $out 2>&1; done
done
ARGCSR_L2PF_AHEAD=4 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "l2_policy or stencil" > gpurun_out/r02_ahead_tests.txt 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/r02_ahead_tests.txt
