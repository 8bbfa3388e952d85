#!/bin/bash
# fp32 pipelined heavy walk: (U, CTAs/SM) = (4,6) default vs (4,5), (5,5), (6,4), (3,4)
mkdir -p gpurun_out; out=gpurun_out/r02_hf32.jsonl; : > $out
for i in 1 2; do
  for v in 0 45 55 64 34; do ARGCSR_HF32=$v timeout 500 python scripts/bench_configs.py C4f32 >> $out 2>&1; done
done
