#!/bin/bash
# Session-3 re-entry check of the restored tree: GPU suite, smoke, default bench, reference arm.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/s3_gputests.txt 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/s3_gputests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/s3_smoke.txt 2>&1; tail -1 gpurun_out/s3_smoke.txt
timeout 1200 python bench.py > gpurun_out/s3_bench.json 2> gpurun_out/s3_bench.err; echo "bench rc=$?"
python - <<'PY'
import json
for f in ("gpurun_out/s3_bench.json",):
    try:
        d = json.loads(open(f).read().splitlines()[-1])
        print(f, d.get("value"), d.get("ms_per_step"), (d.get("roofline") or {}).get("frac"), (d.get("e2e") or {}).get("value"), (d.get("cpu_baseline") or {}).get("value"), d.get("conversion_ms"), d.get("parity"))
        for c in d.get("configs", []):
            print("  ", c["workload"], c.get("ms_per_step"), c["frac"], c.get("conversion_ms"), [(x["impl"], round(x.get("gflops", 0), 1)) for x in c.get("cusparse", [])])
    except Exception as e:
        print(f, "ERR", e)
PY
