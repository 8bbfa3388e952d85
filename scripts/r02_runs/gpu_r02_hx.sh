#!/bin/bash
mkdir -p gpurun_out; out=gpurun_out/r02_hx.jsonl; : > $out
for h in 0 1 2 3 4; do ARGCSR_HEAVY_X=$h timeout 300 python scripts/bench_configs.py C3 C4 >> $out 2>&1; done
cat $out
