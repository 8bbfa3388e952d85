#!/bin/bash
mkdir -p gpurun_out; out=gpurun_out/r02_pl2.jsonl; : > $out
timeout 300 python scripts/bench_configs.py C3 >> $out 2>&1
for t in 3072 4096 1536; do ARGCSR_TILE_THREADS=$t timeout 300 python scripts/bench_configs.py C3 >> $out 2>&1; done
ARGCSR_HEAVY_PIPE=1 timeout 300 python scripts/bench_configs.py C3 >> $out 2>&1
ARGCSR_AUX_PRIO=d timeout 300 python scripts/bench_configs.py C3 >> $out 2>&1
ARGCSR_AUX_PRIO=l timeout 300 python scripts/bench_configs.py C3 >> $out 2>&1
ARGCSR_ULEN=0 timeout 300 python scripts/bench_configs.py C3 >> $out 2>&1
ARGCSR_XPOL=0 timeout 300 python scripts/bench_configs.py C3 >> $out 2>&1
ARGCSR_L2_WINDOW=0 timeout 300 python scripts/bench_configs.py C3 >> $out 2>&1
cat $out
