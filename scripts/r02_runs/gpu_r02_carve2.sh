#!/bin/bash
mkdir -p gpurun_out; out=gpurun_out/r02_carve2.jsonl; : > $out
for c in -1 40 45; do ARGCSR_MAP=0 ARGCSR_CARVEOUT=$c timeout 300 python scripts/bench_configs.py C3 C2 >> $out 2>&1; done
cat $out
