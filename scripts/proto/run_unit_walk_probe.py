"""Unit-walk probe on a synthetic uniform C2 layout: product lane order vs interleaved lanes
(does the warp's x-gather span matter for the register-staged unit walk?)."""
import ctypes
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import workloads  # noqa: E402

lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libgather_probe.so"))
P = ctypes.c_void_p
lib.probe_unit_walk.argtypes = [ctypes.c_int, P, P, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32, P, P, P]


def timeit(fn, n=20, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(n + 1)]
    for i in range(n):
        ev[i].record()
        fn()
    ev[n].record()
    torch.cuda.synchronize()
    return sorted(ev[i].elapsed_time(ev[i + 1]) for i in range(n))[n // 2]


# C2 interior rows: 27 entries, 7 lanes of 4 (last lane 3), groups of 4 rows -> W = 28 lanes, C = 4 steps.
A = workloads.CONFIGS["C2"]["gen"]("cuda")
N = A.num_rows
rp = A.row_pointers
n = rp[1:] - rp[:-1]
R = (N // 4) * 4
G = R // 4
W, C = 28, 4
# element e of row r (e < n_r): lane in row c = e // 4, step j = e % 4 (rows with < 27 entries keep their order)
row = torch.repeat_interleave(torch.arange(N, device="cuda"), n)
e = torch.arange(A.nnz, device="cuda") - rp[row]
keep = row < R
row, e = row[keep], e[keep]
g = row // 4
rl = row % 4
lane = rl * 7 + e // 4
j = e % 4
cols_src = A.columns[keep]
vals_src = A.values[keep]
res = {"rows": R, "groups": G}
x = workloads.bench_input(A.num_cols, "cuda", torch.float64)
out = torch.zeros(1, dtype=torch.float64, device="cuda")
for label in ("product", "interleaved"):
    if label == "product":
        pos_lane = lane
    else:  # stored position p = 4*u' + k holds lane u' + k*W/4
        up, k = lane % (W // 4), lane // (W // 4)
        pos_lane = 4 * up + k
    pos = g * (W * C) + j * W + pos_lane
    cols = torch.full((G * W * C + 8,), -1, dtype=torch.int32, device="cuda")
    vals = torch.zeros(G * W * C + 8, dtype=torch.float64, device="cuda")
    cols[pos] = cols_src
    vals[pos] = vals_src
    for minb in (4, 5):
        ms = timeit(lambda: lib.probe_unit_walk(minb, cols.data_ptr(), vals.data_ptr(), G, W, C, x.data_ptr(),
                                                out.data_ptr(), torch.cuda.current_stream().cuda_stream))
        res[f"{label}_minb{minb}_ms"] = round(ms, 4)
print(json.dumps(res), flush=True)
