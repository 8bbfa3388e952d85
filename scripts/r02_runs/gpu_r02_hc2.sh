#!/bin/bash
mkdir -p gpurun_out; out=gpurun_out/r02_hc2.jsonl; : > $out
for h in 32 48 64 128 250; do ARGCSR_HEAVY_CHUNK=$h timeout 300 python scripts/bench_configs.py C3 >> $out 2>&1; done
cat $out
ARGCSR_HEAVY_CHUNK=64 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "powerlaw" 2>&1 | tail -1
