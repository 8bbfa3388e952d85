#!/bin/bash
mkdir -p gpurun_out; out=gpurun_out/r02_pdl.jsonl; : > $out
for p in 1 0 1 0; do ARGCSR_PDL=$p timeout 300 python scripts/bench_configs.py C2 C3 C4 C4f32 C1 >> $out 2>&1; done
cat $out
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -1
timeout 900 python bench.py --power-iteration --steps 50 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().splitlines()[-1]); print('C5 pdl', d['value'], d['ms_per_step'], d['roofline']['frac'], d['power_iteration']['lambda'])"
ARGCSR_PDL=0 timeout 900 python bench.py --power-iteration --steps 50 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().splitlines()[-1]); print('C5 nopdl', d['value'], d['ms_per_step'], d['roofline']['frac'], d['power_iteration']['lambda'])"
