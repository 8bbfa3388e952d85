#!/bin/bash
# Per-handle L2 policy (regular matrices with x beyond the window: x evict_normal + tile prefetch) vs the previous tree (_ab_head)
mkdir -p gpurun_out; out=gpurun_out/r02_xpol.jsonl; : > $out
for i in 1 2; do
  timeout 500 python scripts/bench_configs.py C5 C3 C2 C4 C4f32 C1 C2:32 | sed 's/"env": {}/"env": {"tree": "new"}/' >> $out 2>&1
  (cd _ab_head && timeout 500 python scripts/bench_configs.py C5 C3 C2 C4 C4f32 C1 C2:32) | sed 's/"env": {}/"env": {"tree": "head"}/' >> $out 2>&1
done
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r02_xpol_tests.txt 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/r02_xpol_tests.txt
timeout 900 python bench.py --power-iteration > gpurun_out/r02_xpol_c5.json 2> gpurun_out/r02_xpol_c5.err; echo "c5 rc=$?"; tail -c 600 gpurun_out/r02_xpol_c5.json
