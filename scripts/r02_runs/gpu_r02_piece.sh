#!/bin/bash
# Tile prefetch piece size per bulk-prefetch instruction (16 KB default vs 2 / 4 / 8 / 64 KB)
mkdir -p gpurun_out; out=gpurun_out/r02_piece.jsonl; : > $out
for i in 1 2; do
  for p in 16384 2048 4096 8192 65536; do ARGCSR_L2PF_PIECE=$p timeout 500 python scripts/bench_configs.py C2 C2:4 C4 C5 >> $out 2>&1; done
done
