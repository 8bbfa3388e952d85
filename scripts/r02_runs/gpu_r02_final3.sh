#!/bin/bash
# Session-3 final tree (columns-only tile prefetch): GPU suite, smoke, default bench (C2 + configs), C5 power iteration, reference arm;
# then ncu (launch list of the default bench command, --set full of the C2/C3/C4/C4f32 SpMV kernels) summarised on the box.
export PYTHONWARNINGS=ignore
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/s3g_gputests.txt 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/s3g_gputests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/s3g_smoke.txt 2>&1; tail -1 gpurun_out/s3g_smoke.txt
timeout 1200 python bench.py > gpurun_out/s3g_bench.json 2> gpurun_out/s3g_bench.err; echo "bench rc=$?"
timeout 1200 python bench.py --power-iteration > gpurun_out/s3g_bench_c5.json 2> gpurun_out/s3g_bench_c5.err; echo "bench c5 rc=$?"
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/s3g_bench_ref.json 2> gpurun_out/s3g_bench_ref.err; echo "ref rc=$?"
TAG=r02e bash scripts/profile_r02.sh > gpurun_out/s3g_profile.log 2>&1; echo "profile rc=$?"; tail -3 gpurun_out/s3g_profile.log
python - <<'PY'
import json
for f in ("gpurun_out/s3g_bench.json", "gpurun_out/s3g_bench_c5.json", "gpurun_out/s3g_bench_ref.json"):
    try:
        d = json.loads(open(f).read().splitlines()[-1])
        print(f, d.get("value"), d.get("ms_per_step"), (d.get("roofline") or {}).get("frac"), (d.get("roofline") or {}).get("traffic"), (d.get("e2e") or {}).get("value"), (d.get("cpu_baseline") or {}).get("value"), d.get("conversion_ms"), d.get("parity"), d.get("clocks"))
        for c in d.get("configs", []):
            print("  ", c["workload"], c.get("ms_per_step"), c["frac"], c.get("conversion_ms"), [(x["impl"], round(x.get("gflops", 0), 1)) for x in c.get("cusparse", [])])
    except Exception as e:
        print(f, "ERR", e)
PY
