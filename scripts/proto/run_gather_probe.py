"""Gather-rate ceiling: a column stream + x gathers (no values, no structure), C3's columns vs synthetic ones."""
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
lib.probe_gather.argtypes = [ctypes.c_int, P, ctypes.c_uint64, P, P, P]
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
    per = sorted(ev[i].elapsed_time(ev[i + 1]) for i in range(n))
    return per[n // 2]


A = workloads.CONFIGS["C3"]["gen"]("cuda")
n = A.nnz
N = A.num_cols
x = workloads.bench_input(N, "cuda", torch.float64)
out = torch.zeros(1, dtype=torch.float64, device="cuda")
g = torch.Generator(device="cuda")
g.manual_seed(1)
streams = {
    "c3_csr": A.columns,
    "uniform_16M": torch.randint(0, N, (n,), device="cuda", generator=g, dtype=torch.int32),
    "uniform_1M": torch.randint(0, 1 << 20, (n,), device="cuda", generator=g, dtype=torch.int32),
    "sequential": (torch.arange(n, device="cuda", dtype=torch.int64) % N).to(torch.int32),
}
# C3 columns sorted inside each 2048-element chunk (line sharing inside a tile)
c = A.columns[: (n // 2048) * 2048].view(-1, 2048)
streams["c3_sorted2048"] = torch.sort(c, dim=1).values.flatten().contiguous()
streams["c3_shuffled"] = A.columns[torch.randperm(n, device="cuda", generator=g)]
deg = torch.bincount(A.columns.long(), minlength=N)
order = torch.argsort(-deg, stable=True)
newidx = torch.empty_like(order)
newidx[order] = torch.arange(N, device="cuda")
streams["c3_degree_rank"] = newidx[A.columns.long()].to(torch.int32)
# octave ranks (the product's x remap): floor(log2 deg) descending, index order within an octave
octv = torch.where(deg > 0, torch.floor(torch.log2(deg.clamp(min=1).double())), torch.full_like(deg, -1, dtype=torch.float64))
order2 = torch.argsort(-octv, stable=True)
newidx2 = torch.empty_like(order2)
newidx2[order2] = torch.arange(N, device="cuda")
streams["c3_octave_rank"] = newidx2[A.columns.long()].to(torch.int32)
for name in ("c3_csr", "c3_shuffled", "c3_degree_rank", "c3_octave_rank"):
    cols = streams[name].contiguous()
    res = {"flat_spmv": name}
    for v in (0, 1, 2):
        ms = timeit(lambda: lib.probe_spmv_flat(v, cols.data_ptr(), A.values.data_ptr(), n, x.data_ptr(),
                                                out.data_ptr(), torch.cuda.current_stream().cuda_stream))
        res[f"v{v}_ms"] = round(ms, 4)
        res[f"v{v}_frac"] = round((n * 12 + 2 * N * 8) / ms / 1e6 / 6538.3, 4)
    print(json.dumps(res), flush=True)
if os.environ.get("FLAT_ONLY"):
    sys.exit(0)
for name, cols in streams.items():
    cols = cols.contiguous()
    nn = cols.numel()
    res = {"stream": name, "n": nn}
    for v in (0, 1, 2, 3, 4, 5, 6, 7):
        ms = timeit(lambda: lib.probe_gather(v, cols.data_ptr(), nn, x.data_ptr(), out.data_ptr(),
                                             torch.cuda.current_stream().cuda_stream))
        res[f"v{v}_ms"] = round(ms, 4)
        res[f"v{v}_Ggps"] = round(nn / ms / 1e6, 1)
    print(json.dumps(res), flush=True)
