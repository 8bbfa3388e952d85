#!/bin/bash
mkdir -p gpurun_out; out=gpurun_out/r02_tt.jsonl; : > $out
for t in 512 448 480 416 384 576 640; do ARGCSR_TILE_THREADS=$t timeout 300 python scripts/bench_configs.py C2 >> $out 2>&1; done
cat $out
