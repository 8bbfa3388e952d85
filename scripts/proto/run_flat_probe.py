"""Structure-free SpMV ceiling per config: stream columns + values, gather x, no row sums (scripts/proto/gather_probe.cu)."""
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


for name in sys.argv[1:]:
    A = workloads.CONFIGS[name]["gen"]("cuda")
    x = workloads.bench_input(A.num_cols, "cuda", torch.float64)
    out = torch.zeros(1, dtype=torch.float64, device="cuda")
    n = A.nnz
    res = {"config": name, "nnz": n}
    for v in (0, 1, 2):
        ms = timeit(lambda: lib.probe_spmv_flat(v, A.columns.data_ptr(), A.values.data_ptr(), n, x.data_ptr(),
                                                out.data_ptr(), torch.cuda.current_stream().cuda_stream))
        res[f"v{v}_ms"] = round(ms, 4)
        res[f"v{v}_frac"] = round((n * 12 + (A.num_rows + A.num_cols) * 8) / ms / 1e6 / 6538.3, 4)
    print(json.dumps(res), flush=True)
    del A, x
    torch.cuda.empty_cache()
