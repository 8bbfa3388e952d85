# PAIR kernel (every light chunk <= 2): parity + A/B
export PYTHONWARNINGS=ignore
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_multigpu_device.py tests/test_peer.py -m gpu -x -q 2>&1 | tail -3
for c in C1 C4 C4f32 C2; do
 for p in 1 0; do
  ARGCSR_PAIR=$p timeout 300 python bench.py --config $c --steps 100 --warmup 5 --no-variants --no-cpu-baseline 2>gpurun_out/err_$c_$p.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c pair=$p', round(d['ms_per_step'],4), d['value'], d['roofline']['frac'])" || tail -3 gpurun_out/err_$c_$p.txt
 done
done
