#!/bin/bash
# Lane walks prefetch their next batch of element steps into L2 (ARGCSR_SWPF bit 0 heavy, bit 1 light) vs off
mkdir -p gpurun_out; out=gpurun_out/r02_swpf.jsonl; : > $out
for i in 1 2; do
  for v in 0 1 2 3; do ARGCSR_SWPF=$v timeout 400 python scripts/bench_configs.py C4 C4f32 C3 C2:32 C2:4 >> $out 2>&1; done
done
ARGCSR_SWPF=3 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r02_swpf_tests.txt 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/r02_swpf_tests.txt
