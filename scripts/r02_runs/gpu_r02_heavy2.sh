#!/bin/bash
mkdir -p gpurun_out; out=gpurun_out/r02_heavy2.jsonl; : > $out
for h in 0 1; do ARGCSR_HEAVY2=$h timeout 300 python scripts/bench_configs.py C4 C4f32 C3 C4:4 >> $out 2>&1; done
cat $out
ARGCSR_HEAVY2=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_multigpu_device.py tests/test_peer.py -q -x -p no:cacheprovider -k "heavy or powerlaw or dense or norm or fused or fp32 or peer" 2>&1 | tail -1
