#!/bin/bash
# Light/heavy boundary sweep on C3 (power-law): groups with chunk > H on the lane-walk heavy path.
mkdir -p gpurun_out; out=gpurun_out/r02_hchunk.jsonl; : > $out
for h in 16 8 4 2; do
for p in 0 4 8; do
if [ $p = 0 ]; then ARGCSR_HEAVY_CHUNK=$h timeout 300 python scripts/bench_configs.py C3 >> $out 2>&1
else ARGCSR_HEAVY_CHUNK=$h ARGCSR_HEAVY_PIPE=$p timeout 300 python scripts/bench_configs.py C3 >> $out 2>&1; fi
done; done


cat $out
