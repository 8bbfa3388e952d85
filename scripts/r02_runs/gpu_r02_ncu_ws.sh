#!/bin/bash
# ncu --set full of the ws kernel on C2 (one launch), plus the default light kernel for comparison.
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:spmv_ws -s 3 -c 1 -o gpurun_out/r02_ncu_ws_C2 \
    python scripts/bench_configs.py C2 > gpurun_out/r02_ncu_ws_C2.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/r02_ncu_ws_C2.log
python scripts/ncu_summary.py gpurun_out/r02_ncu_ws_C2.ncu-rep 40 > gpurun_out/r02_ncu_ws_C2.txt 2>&1
cat gpurun_out/r02_ncu_ws_C2.txt | head -80
