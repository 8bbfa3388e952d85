# unit-length table: parity (forced on/off) + A/B on C1-C4
export PYTHONWARNINGS=ignore
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "unit_lengths or powerlaw or corpus_grid or host_staged or stencil" 2>&1 | tail -4
for c in C3:1 C4:1 C2:1 C1:1 C2:32; do
  cfg=${c%%:*}; d=${c##*:}
  for u in 1 0; do
    ARGCSR_ULEN=$u timeout 300 python bench.py --config $cfg --dcs $d --steps 50 --warmup 5 --no-variants --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg dcs=$d ulen=$u', round(d['ms_per_step'],4), d['roofline']['frac'], 'ulenB', d['format'].get('unit_len_bytes'))"
  done
done
ARGCSR_SPMV_VARIANT=F4P0B5 timeout 300 python bench.py --config C3 --steps 50 --warmup 5 --no-variants --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C3 FLAT', round(d['ms_per_step'],4), d['roofline']['frac'])"
ARGCSR_SPMV_VARIANT=F4P0B5 timeout 300 python bench.py --config C1 --steps 50 --warmup 5 --no-variants --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C1 FLAT', round(d['ms_per_step'],4), d['roofline']['frac'])"
