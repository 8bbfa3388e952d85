#!/bin/bash
# Full GPU suite, smoke, default bench, power-iteration bench (C5), launch list + ncu of the default C2 step.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r02f_gputests.txt 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/r02f_gputests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02f_smoke.txt 2>&1; tail -1 gpurun_out/r02f_smoke.txt
timeout 1200 python bench.py > gpurun_out/r02f_bench.json 2> gpurun_out/r02f_bench.err; echo "bench rc=$?"
timeout 1200 python bench.py --power-iteration > gpurun_out/r02f_bench_c5.json 2> gpurun_out/r02f_bench_c5.err; echo "bench c5 rc=$?"
python - <<'PY'
import json
for f in ("gpurun_out/r02f_bench.json", "gpurun_out/r02f_bench_c5.json"):
    try:
        d = json.loads(open(f).read().splitlines()[-1])
        print(f, d["value"], d["ms_per_step"], d["roofline"]["frac"], d.get("e2e", {}).get("value"), d.get("cpu_baseline", {}).get("value"), d.get("conversion_ms"), d.get("parity"))
        for c in d.get("configs", []):
            print("  ", c["workload"], c.get("ms_per_step"), c["frac"], [(x["impl"], round(x.get("gflops", 0), 1)) for x in c.get("cusparse", [])])
    except Exception as e:
        print(f, "ERR", e)
PY
