#!/bin/bash
# Tile prefetch pieces issued by lane 0 only (ARGCSR_L2PF_ONE) vs spread over the warp's lanes
mkdir -p gpurun_out; out=gpurun_out/r02_onelane.jsonl; : > $out
for i in 1 2 3; do
  timeout 500 python scripts/bench_configs.py C2 C2:4 C4 C5 >> $out 2>&1
  ARGCSR_L2PF_ONE=1 timeout 500 python scripts/bench_configs.py C2 C2:4 C4 C5 >> $out 2>&1
done
