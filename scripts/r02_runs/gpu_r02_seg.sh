#!/bin/bash
# fp32 heavy lanes as K j-segments (ARGCSR_HEAVY_SEG): parity tests, then A/B on C4 fp32 (K=2 default vs 1), C4/C3 fp64 unchanged
mkdir -p gpurun_out; out=gpurun_out/r02_seg.jsonl; : > $out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "fp32 or dense_rows or heavy" > gpurun_out/r02_seg_tests.txt 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/r02_seg_tests.txt
for i in 1 2 3; do
  timeout 300 python scripts/bench_configs.py C4f32 >> $out 2>&1
  ARGCSR_HEAVY_SEG=1 timeout 300 python scripts/bench_configs.py C4f32 >> $out 2>&1
done
timeout 300 python scripts/bench_configs.py C4 C3 >> $out 2>&1
cat $out
