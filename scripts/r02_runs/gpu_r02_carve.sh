#!/bin/bash
# shared-memory carve-out sweep (more L1 for the x gathers)
mkdir -p gpurun_out; out=gpurun_out/r02_carve.jsonl; : > $out
for c in 30 35 40 45 60; do ARGCSR_CARVEOUT=$c timeout 300 python scripts/bench_configs.py C3 C2 C4 >> $out 2>&1; done
cat $out
