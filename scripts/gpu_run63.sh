# final: full GPU suite, smoke, C3 bench with DYN default
export PYTHONWARNINGS=ignore
timeout 2400 python -m pytest tests/ -m gpu -x -q 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
mkdir -p gpurun_out/bench
timeout 900 python bench.py --config C3 > gpurun_out/bench/bench_C3.json 2>/dev/null; tail -c 300 gpurun_out/bench/bench_C3.json
