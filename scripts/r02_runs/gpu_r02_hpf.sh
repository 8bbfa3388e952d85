#!/bin/bash
# Long-chunk groups: the first lane bulk-prefetches the group's element-step rows ARGCSR_HEAVY_PF steps ahead; vs the previous tree (_ab_head)
mkdir -p gpurun_out; out=gpurun_out/r02_hpf.jsonl; : > $out
for i in 1 2; do
  (cd _ab_head && timeout 500 python scripts/bench_configs.py C4 C4f32 C3) | sed 's/"env": {}/"env": {"tree": "head"}/' >> $out 2>&1
  for d in 0 16 32 64; do ARGCSR_HEAVY_PF=$d timeout 500 python scripts/bench_configs.py C4 C4f32 C3 >> $out 2>&1; done
done
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "l2_policy or dense_rows or powerlaw" > gpurun_out/r02_hpf_tests.txt 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/r02_hpf_tests.txt
