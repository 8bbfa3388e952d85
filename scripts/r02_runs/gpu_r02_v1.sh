#!/bin/bash
mkdir -p gpurun_out; out=gpurun_out/r02_v1.jsonl; : > $out
export ARGCSR_VEC=1 ARGCSR_TILE_THREADS=2048
for u in 0 8 6 3; do ARGCSR_V1U=$u timeout 300 python scripts/bench_configs.py C3 >> $out 2>&1; done
ARGCSR_LIGHT_DYN=0 timeout 300 python scripts/bench_configs.py C3 >> $out 2>&1
ARGCSR_MAP=0 timeout 300 python scripts/bench_configs.py C3 >> $out 2>&1
ARGCSR_TILE_THREADS=1024 timeout 300 python scripts/bench_configs.py C3 >> $out 2>&1
timeout 300 python scripts/bench_configs.py C2:32 C4 C4f32 >> $out 2>&1
unset ARGCSR_VEC ARGCSR_TILE_THREADS
timeout 300 python scripts/bench_configs.py C3 >> $out 2>&1
cat $out
