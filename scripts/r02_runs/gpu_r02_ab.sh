#!/bin/bash
# A/B on one box: C2/C3/C4 timings of the tree at bbcd788 (scripts/proto/old) vs HEAD.
mkdir -p gpurun_out
for i in 1 2; do
timeout 300 python scripts/proto/old/scripts/bench_configs.py C2 C3 C4 > gpurun_out/r02_ab_old$i.jsonl 2>&1
timeout 300 python scripts/bench_configs.py C2 C3 C4 > gpurun_out/r02_ab_new$i.jsonl 2>&1
done
ARGCSR_HEAVY_BLOCKED=0 timeout 300 python scripts/bench_configs.py C2 C3 C4 > gpurun_out/r02_ab_new_lw.jsonl 2>&1
head -50 gpurun_out/r02_ab_*.jsonl
