#!/bin/bash
# Tile prefetch end rounded down (never past the array): GPU suite + C2 bench_configs
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r02_bounds_tests.txt 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/r02_bounds_tests.txt
timeout 500 python scripts/bench_configs.py C2 C2:4 C5 C4 > gpurun_out/r02_bounds.jsonl 2>&1; cut -c1-100 gpurun_out/r02_bounds.jsonl
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
