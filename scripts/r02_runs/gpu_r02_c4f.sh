#!/bin/bash
mkdir -p gpurun_out; out=gpurun_out/r02_c4f.jsonl; : > $out
for h in 0 7 8 9; do ARGCSR_HEAVY_X=$h timeout 300 python scripts/bench_configs.py C4f32 >> $out 2>&1; done
cat $out
