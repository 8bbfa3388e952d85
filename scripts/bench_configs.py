"""Quick per-config SpMV timings on one GPU (no parity leg): C2, C3, C4, C4f32
with the current defaults; prints one JSON object per config.  Experiment
switches (ARGCSR_*) come from the environment."""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1203_5737_b200 as argcsr  # noqa: E402
import workloads  # noqa: E402

PEAK = 6538.3
names = sys.argv[1:] or ["C2", "C3", "C4", "C4f32"]
for name in names:
    tpg, dcs = 128, 1
    if ":" in name:
        name, dcs = name.split(":")
        dcs = int(dcs)
    cfg = workloads.CONFIGS[name]
    dt = torch.float64 if cfg["dtype"] == "float64" else torch.float32
    sv = 8 if dt == torch.float64 else 4
    A = cfg["gen"]("cuda")
    vals = A.values.to(dt)
    torch.cuda.synchronize()
    m = argcsr.argcsr_from_torch(A.num_rows, A.num_cols, A.row_pointers, A.columns, vals, tpg, dcs)
    x = workloads.bench_input(A.num_cols, "cuda", dt)
    y = torch.empty(A.num_rows, dtype=dt, device="cuda")
    st = torch.cuda.current_stream()
    for _ in range(5):
        m.spmv_device(x.data_ptr(), y.data_ptr(), st.cuda_stream)
    torch.cuda.synchronize()
    n = 30
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(n + 1)]
    for i in range(n):
        ev[i].record()
        m.spmv_device(x.data_ptr(), y.data_ptr(), st.cuda_stream)
    ev[n].record()
    torch.cuda.synchronize()
    per = [ev[i].elapsed_time(ev[i + 1]) for i in range(n)]
    ms = ev[0].elapsed_time(ev[n]) / n
    ab = A.nnz * (sv + 4) + (A.num_rows + A.num_cols) * sv
    print(json.dumps({"config": name, "dcs": dcs, "ms": round(ms, 4), "median_ms": round(statistics.median(per), 4),
                      "gflops": round(2 * A.nnz / ms / 1e6, 1), "frac": round(ab / ms / 1e6 / PEAK, 4),
                      "heavy": m.heavy_groups, "tiles": m.light_tiles, "x_remap": m.x_remap,
                      "env": {k: v for k, v in os.environ.items() if k.startswith("ARGCSR_")}}), flush=True)
    m.free()
    del m, A, vals, x, y
    torch.cuda.empty_cache()
