"""Prototype timing: row-stream tile kernel + long-row kernel vs the product SpMV (C2/C3/C4 fp64)."""
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

lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libstream_proto.so"))
P = ctypes.c_void_p
lib.proto_tile.argtypes = [ctypes.c_int, P, P, P, P, P, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32, P, P, P]
lib.proto_long.argtypes = [ctypes.c_int, P, P, P, P, P, P, ctypes.c_uint32, ctypes.c_uint32, P, P, P]
PEAK = 6538.3


def timeit(fn, n=30, warm=5):
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


def run(name, E, LMAX, tile_variants=(1, 5, 6, 7, 8, 9), long_variants=(0,)):
    cfg = workloads.CONFIGS[name]
    A = cfg["gen"]("cuda")
    N = A.num_rows
    rp = A.row_pointers
    m = argcsr.argcsr_from_torch(N, A.num_cols, rp, A.columns, A.values, 128, 1)
    x = workloads.bench_input(A.num_cols, "cuda", torch.float64)
    y_ref = torch.empty(N, dtype=torch.float64, device="cuda")
    st = torch.cuda.current_stream()
    m.spmv_device(x.data_ptr(), y_ref.data_ptr(), st.cuda_stream)
    t_prod = timeit(lambda: m.spmv_device(x.data_ptr(), y_ref.data_ptr(), st.cuda_stream))
    tm = torch.from_numpy(np.asarray(m.threads_mapping).astype(np.int64)).cuda()
    first = torch.from_numpy(np.array([g.first_row for g in m.groups], dtype=np.int64)).cuda()
    isfirst = torch.zeros(N, dtype=torch.bool, device="cuda")
    isfirst[first] = True
    prev = torch.cat([torch.zeros(1, dtype=torch.int64, device="cuda"), tm[:-1]])
    t = torch.where(isfirst, tm, tm - prev)
    n = rp[1:] - rp[:-1]
    islong = n > LMAX
    # short stream
    keep = torch.repeat_interleave(~islong, n)
    scols = A.columns[keep]
    svals = A.values[keep]
    pad = 8
    scols = torch.cat([scols, torch.zeros(pad, dtype=torch.int32, device="cuda")])
    svals = torch.cat([svals, torch.zeros(pad, dtype=torch.float64, device="cuda")])
    sn = torch.where(islong, 0, n)
    srp = torch.zeros(N + 1, dtype=torch.int64, device="cuda")
    srp[1:] = torch.cumsum(sn, 0)
    snnz = int(srp[-1])
    tt = (t | (islong.to(torch.int64) << 15)).to(torch.int32).to(torch.int16)
    nt0 = (snnz + E - 1) // E
    keys = torch.arange(nt0 + 1, device="cuda", dtype=torch.int64) * E
    tr0 = torch.searchsorted(srp[:N].contiguous(), keys, right=False)
    tiles = {}
    for rc in (256, 512):
        b = torch.unique(torch.cat([tr0, torch.arange(0, N, rc, device="cuda"), torch.tensor([N], device="cuda")]))
        b = b[b <= N]
        # split any tile still above rc rows
        tiles[rc] = b.to(torch.int32).contiguous()
        assert int((b[1:] - b[:-1]).max()) <= rc
    srp32 = srp.to(torch.int32)
    # long region
    lrows = torch.nonzero(islong).flatten()
    L = lrows.numel()
    lkeep = torch.repeat_interleave(islong, n)
    lcols = A.columns[lkeep].contiguous()
    lvals = A.values[lkeep].contiguous()
    ln = n[lrows]
    lrp = torch.zeros(L + 1, dtype=torch.int64, device="cuda")
    lrp[1:] = torch.cumsum(ln, 0)
    lt = t[lrows].to(torch.int32).to(torch.int16)
    order = torch.argsort(ln, descending=True, stable=True).to(torch.int32)
    maxt = int(t[lrows].max()) if L else 1
    lrow32 = lrows.to(torch.int32)
    cap = E + LMAX + 8
    y = torch.full((N,), float("nan"), dtype=torch.float64, device="cuda")
    s1 = torch.cuda.Stream(priority=-1)
    res = {"config": name, "E": E, "LMAX": LMAX, "long_rows": L, "long_nnz": int(lrp[-1]), "short_nnz": snnz,
           "ntiles": tiles[256].numel() - 1, "product_ms": round(t_prod, 4), "product_frac": None}
    ab = A.nnz * 12 + (N + A.num_cols) * 8
    res["product_frac"] = round(ab / t_prod / 1e6 / PEAK, 4)

    def tile(v):
        rc = 512 if v in (8, 9) else 256
        tr = tiles[rc]
        return lambda: lib.proto_tile(v, svals.data_ptr(), scols.data_ptr(), srp32.data_ptr(), tt.data_ptr(),
                                      tr.data_ptr(), tr.numel() - 1, cap, rc, x.data_ptr(), y.data_ptr(),
                                      torch.cuda.current_stream().cuda_stream)

    def lng(v, stream=None):
        return lambda: lib.proto_long(v, lvals.data_ptr(), lcols.data_ptr(), lrp.data_ptr(), lt.data_ptr(),
                                      lrow32.data_ptr(), order.data_ptr(), L, maxt, x.data_ptr(), y.data_ptr(),
                                      (stream or torch.cuda.current_stream()).cuda_stream)

    for v in tile_variants:
        res[f"tile{v}_ms"] = round(timeit(tile(v)), 4)
    for v in long_variants:
        if L:
            res[f"long{v}_ms"] = round(timeit(lng(v)), 4)
    bt = min([v for v in tile_variants if v not in (4, 5)], key=lambda v: res[f"tile{v}_ms"])
    for v in tile_variants:
        if v in (4, 5):
            continue
        y.fill_(float("nan"))
        tile(v)()
        if L:
            lng(long_variants[0])()
        torch.cuda.synchronize()
        res[f"tile{v}_exact"] = bool(torch.equal(y, y_ref))
    bl = min(long_variants, key=lambda v: res.get(f"long{v}_ms", 0))

    def both():
        if L:
            ev = torch.cuda.Event()
            ev.record()
            s1.wait_event(ev)
            lng(bl, s1)()
        tile(bt)()
        if L:
            ev2 = torch.cuda.Event()
            ev2.record(s1)
            torch.cuda.current_stream().wait_event(ev2)

    y.fill_(float("nan"))
    both()
    torch.cuda.synchronize()
    res["bit_exact"] = bool(torch.equal(y, y_ref))
    if not res["bit_exact"]:
        bad = torch.nonzero(y != y_ref).flatten()
        res["mismatch"] = int(bad.numel())
        res["first_bad"] = [int(bad[0]), float(y[bad[0]]), float(y_ref[bad[0]]), int(n[bad[0]]), int(t[bad[0]])]
    tb = timeit(both)
    res["both_ms"] = round(tb, 4)
    res["both_frac"] = round(ab / tb / 1e6 / PEAK, 4)
    res["both_gflops"] = round(2 * A.nnz / tb / 1e6, 1)
    print(json.dumps(res), flush=True)
    m.free()


if __name__ == "__main__":
    for spec in sys.argv[1:]:
        name, E, LMAX = spec.split(":")
        run(name, int(E), int(LMAX))
