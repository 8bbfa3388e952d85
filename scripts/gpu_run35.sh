# C3 light-kernel limiter analysis: one --set full capture (raw page + source) + window on/off
export PYTHONWARNINGS=ignore
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:spmv_light -s 3 -c 1 \
    -o gpurun_out/c3_light_full python bench.py --config C3 --steps 3 --warmup 3 --no-variants --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out/
for w in 1 0; do ARGCSR_L2_WINDOW=$w timeout 300 python bench.py --config C3 --steps 30 --warmup 5 --no-variants --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('window=$w', d['ms_per_step'], d['roofline']['frac'])"; done
