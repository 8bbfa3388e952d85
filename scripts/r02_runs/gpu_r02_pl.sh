#!/bin/bash
mkdir -p gpurun_out; out=gpurun_out/r02_pl.jsonl; : > $out
timeout 300 python scripts/bench_configs.py C3 C2 C4 C4f32 C2:32 >> $out 2>&1
cat $out
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
