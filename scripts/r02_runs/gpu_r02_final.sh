#!/bin/bash
# Final tree: full GPU suite, smoke, default bench (C2 + configs), C5 power iteration, ncu of the C3 kernels.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r02z_gputests.txt 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/r02z_gputests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02z_smoke.txt 2>&1; tail -1 gpurun_out/r02z_smoke.txt
timeout 1200 python bench.py > gpurun_out/r02z_bench.json 2> gpurun_out/r02z_bench.err; echo "bench rc=$?"
timeout 1200 python bench.py --power-iteration > gpurun_out/r02z_bench_c5.json 2> gpurun_out/r02z_bench_c5.err; echo "bench c5 rc=$?"
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/r02z_bench_ref.json 2> gpurun_out/r02z_bench_ref.err; echo "ref rc=$?"
TAG=r02c
ncu --set full --clock-control none --import-source on -k regex:spmv_ -s 6 -c 2 -o gpurun_out/${TAG}_full_C3_dcs1_compact \
    python bench.py --config C3 --steps 5 --warmup 3 --no-variants --no-cpu-baseline --no-configs > /dev/null 2>&1
python scripts/summarize_profiles.py $TAG > /dev/null 2>&1
mkdir -p gpurun_out/prof_out && cp profiles/${TAG}_* profiles/ncu_traffic.json gpurun_out/prof_out/ 2>/dev/null
rm -f gpurun_out/*.ncu-rep
python - <<'PY'
import json
for f in ("gpurun_out/r02z_bench.json", "gpurun_out/r02z_bench_c5.json", "gpurun_out/r02z_bench_ref.json"):
    try:
        d = json.loads(open(f).read().splitlines()[-1])
        print(f, d.get("value"), d.get("ms_per_step"), (d.get("roofline") or {}).get("frac"), (d.get("e2e") or {}).get("value"), (d.get("cpu_baseline") or {}).get("value"), d.get("conversion_ms"), d.get("parity"))
        for c in d.get("configs", []):
            print("  ", c["workload"], c.get("ms_per_step"), c["frac"], c.get("conversion_ms"), [(x["impl"], round(x.get("gflops", 0), 1)) for x in c.get("cusparse", [])])
    except Exception as e:
        print(f, "ERR", e)
PY
