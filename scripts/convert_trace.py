"""Per-phase conversion timings (ARGCSR_TRACE=1) of the BASELINE configs, twice each."""
import os
import sys
import time

os.environ.setdefault("ARGCSR_TRACE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1203_5737_b200 as argcsr  # noqa: E402
import workloads  # noqa: E402

for name in sys.argv[1:] or ["C2", "C3", "C4"]:
    cfg = workloads.CONFIGS[name]
    A = cfg["gen"]("cuda")
    dt = torch.float64 if cfg["dtype"] == "float64" else torch.float32
    vals = A.values.to(dt)
    for rep in range(2):
        torch.cuda.synchronize()
        t = time.perf_counter()
        m = argcsr.argcsr_from_torch(A.num_rows, A.num_cols, A.row_pointers, A.columns, vals, 128, 1)
        torch.cuda.synchronize()
        print(f"{name} rep{rep}: {1e3 * (time.perf_counter() - t):.1f} ms  groups={m.num_groups} heavy={m.heavy_groups}"
              f" remap={m.x_remap}", file=sys.stderr, flush=True)
        m.free()
        del m
    del A, vals
    torch.cuda.empty_cache()
