#!/bin/bash
mkdir -p gpurun_out; out=gpurun_out/r02_c1.jsonl; : > $out
for t in 512 384 256 192 128; do ARGCSR_TILE_THREADS=$t timeout 300 python scripts/bench_configs.py C1 >> $out 2>&1; done
ARGCSR_PAIR=0 timeout 300 python scripts/bench_configs.py C1 >> $out 2>&1
ARGCSR_PAIR=0 ARGCSR_TILE_THREADS=256 timeout 300 python scripts/bench_configs.py C1 >> $out 2>&1
cat $out
