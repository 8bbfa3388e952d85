"""Structure-free probe on the STORED (lane-compact, j-major) order vs CSR order:
is the C2/C3 gap to the probe the gather pattern of the ARG-CSR layout or the
kernel structure (tiles, metadata, barriers, row sums)?"""
import ctypes
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_1203_5737_b200 as argcsr  # noqa: E402
import workloads  # noqa: E402

lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libgather_probe.so"))
P = ctypes.c_void_p
lib.probe_spmv_flat.argtypes = [ctypes.c_int, P, P, ctypes.c_uint64, P, P, P]


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


def compact_order(A, m, V=4):
    """Positions of the CSR entries in the lane-compact j-major layout (light groups only, heavy ignored)."""
    dev = "cuda"
    N = A.num_rows
    rp = A.row_pointers
    n = (rp[1:] - rp[:-1])
    tm = torch.from_numpy(np.asarray(m.threads_mapping).astype(np.int64)).to(dev)
    G = np.asarray(m.groups_array).reshape(-1, 4) if hasattr(m, "groups_array") else None
    first = torch.from_numpy(G[:, 0].astype(np.int64)).to(dev)
    chunk = torch.from_numpy(G[:, 3].astype(np.int64)).to(dev)
    ng = first.numel()
    isfirst = torch.zeros(N, dtype=torch.bool, device=dev)
    isfirst[first] = True
    gid = torch.cumsum(isfirst.to(torch.int64), 0) - 1
    prev = torch.cat([torch.zeros(1, dtype=torch.int64, device=dev), tm[:-1]])
    lane0 = torch.where(isfirst, torch.zeros_like(tm), prev)  # first lane of the row in its group
    t = tm - lane0
    last = torch.cat([first[1:] - 1, torch.tensor([N - 1], device=dev)])
    assigned = tm[last]
    stride = (assigned + V - 1) // V * V
    gsl = chunk * stride
    goff = torch.cumsum(gsl, 0) - gsl
    # per entry: row, local index i, lane c (ceil-first split), j
    row = torch.repeat_interleave(torch.arange(N, device=dev), n)
    i = torch.arange(A.nnz, device=dev) - rp[row]
    nr, tr = n[row], t[row]
    base, extra = nr // tr, nr % tr
    big = extra * (base + 1)
    c = torch.where(i < big, i // (base + 1), extra + (i - big) // torch.clamp(base, min=1))
    j = torch.where(i < big, i % (base + 1), (i - big) % torch.clamp(base, min=1))
    g = gid[row]
    pos = goff[g] + j * stride[g] + lane0[row] + c
    total = int(gsl.sum())
    return pos, total


for name in sys.argv[1:]:
    A = workloads.CONFIGS[name]["gen"]("cuda")
    m = argcsr.argcsr_from_torch(A.num_rows, A.num_cols, A.row_pointers, A.columns, A.values, 128, 1)
    pos, total = compact_order(A, m)
    cols = torch.zeros(total + 8, dtype=torch.int32, device="cuda")   # padding gathers x[0] (one hot line)
    vals = torch.zeros(total + 8, dtype=torch.float64, device="cuda")
    cols[pos] = A.columns
    vals[pos] = A.values
    x = workloads.bench_input(A.num_cols, "cuda", torch.float64)
    out = torch.zeros(1, dtype=torch.float64, device="cuda")
    res = {"config": name, "nnz": A.nnz, "stored": total}
    for label, cc, vv, nn in (("csr", A.columns, A.values, A.nnz), ("compact", cols, vals, total)):
        ms = timeit(lambda: lib.probe_spmv_flat(0, cc.data_ptr(), vv.data_ptr(), nn, x.data_ptr(), out.data_ptr(),
                                                torch.cuda.current_stream().cuda_stream))
        res[f"{label}_ms"] = round(ms, 4)
    print(json.dumps(res), flush=True)
    m.free()
    del A, cols, vals, pos
    torch.cuda.empty_cache()
