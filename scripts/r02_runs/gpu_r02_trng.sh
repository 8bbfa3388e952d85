#!/bin/bash
# Tile L2 prefetch issued from precomputed per-tile ranges (this tree) vs from the group descriptors (_ab_head = previous commit)
mkdir -p gpurun_out; out=gpurun_out/r02_trng.jsonl; : > $out
for i in 1 2 3; do
  timeout 400 python scripts/bench_configs.py C2 C2:4 C1 C4 | sed 's/"env": {/"env": {"tree": "new", /' >> $out 2>&1
  (cd _ab_head && timeout 400 python scripts/bench_configs.py C2 C2:4 C1 C4) | sed 's/"env": {/"env": {"tree": "head", /' >> $out 2>&1
done
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r02_trng_tests.txt 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/r02_trng_tests.txt
