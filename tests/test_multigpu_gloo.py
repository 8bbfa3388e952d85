"""The multi-GPU layer's host logic on CPU with the gloo
backend, world size 2: nnz-balanced row split, per-slice conversion (each
slice equals the reference conversion of that slice), the all-gather of y
slices (even and uneven splits) and the power iteration with its fused
normalisation, against a single-process CPU run of the same algorithm.  The
per-rank engine here is the oracle (test-only); on the GPU it is the CUDA
path (tests/test_multigpu_device.py)."""
import os
import sys
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parent.parent


class OracleEngine:
    """CPU stand-in for DeviceEngine: the oracle's conversion and SpMV of the slice."""

    def __init__(self, sl, tpg, dcs):
        import oracle

        self.orc = oracle.orc()
        self.device = torch.device("cpu")
        self.csr = oracle.Csr(sl.num_rows, sl.num_cols, np.asarray(sl.row_pointers, np.uint64),
                              np.asarray(sl.columns, np.int32), np.asarray(sl.values, np.float64))
        self.m = self.orc.argcsr_from_csr(self.csr, tpg, dcs)

    def spmv(self, x, y, x_scale=None):
        xv = x.numpy()
        if x_scale is not None:
            xv = xv * x_scale.numpy()[0]
        y.copy_(torch.from_numpy(self.orc.spmv_argcsr(self.m, xv)))

    @property
    def num_groups(self):
        return int(self.m.groups.shape[0])

    def group_first_rows(self):
        return np.concatenate([self.m.groups[:, 0], [self.m.num_rows]]).astype(np.int64)

    def spmv_range(self, x, y, g0, g1, x_scale=None, reuse_x=False):
        """Rows of groups [g0, g1) only (spmv_argcsr_groups semantics)."""
        if g1 <= g0:
            return
        xv = x.numpy()
        if x_scale is not None:
            xv = xv * x_scale.numpy()[0]
        full = self.orc.spmv_argcsr(self.m, xv)
        a = int(self.m.groups[g0, 0])
        b = int(self.m.groups[g1, 0]) if g1 < self.num_groups else self.m.num_rows
        y[a:b] = torch.from_numpy(full[a:b])


def reference_power_iteration(A, x0, iters, tpg, dcs):
    """Single-process CPU run of the same algorithm (oracle SpMV, sequential norm)."""
    import oracle

    orc = oracle.orc()
    M = orc.argcsr_from_csr(A, tpg, dcs)
    x, scale, s2 = x0.copy(), 1.0, 0.0
    for _ in range(iters):
        y = orc.spmv_argcsr(M, x * scale)
        s2 = float(np.dot(y, y))
        x = y
        scale = 1.0 / np.sqrt(s2)
    return float(np.sqrt(s2)), x * scale


def _matrix(kind):
    sys.path.insert(0, str(ROOT / "tests"))
    from helpers import powerlaw_csr, stencil27

    if kind == "stencil":
        return stencil27(9)  # 729 rows: uneven split -> per-owner broadcasts
    if kind == "stencil8":
        return stencil27(8)  # 512 rows: even split -> one all_gather_into_tensor
    return powerlaw_csr(3001, 3001, seed=4, heavy_rows=[(7, 2000)])


def _worker(rank, world, port, kind, tpg, dcs, iters, out, overlap, exchange="auto"):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, str(ROOT))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_1203_5737_b200.multigpu import DistributedArgCsr

        A = _matrix(kind)
        D = DistributedArgCsr(A.num_rows, A.num_cols, A.row_pointers, A.columns, A.values, tpg, dcs,
                              engine_factory=lambda sl: OracleEngine(sl, tpg, dcs), overlap=overlap,
                              exchange=exchange)
        # the slice's conversion equals the reference conversion of the slice
        sl = D.slice
        want = oracle.orc().argcsr_from_csr(D.engine.csr, tpg, dcs)
        assert np.array_equal(D.engine.m.groups, want.groups)
        x0 = torch.from_numpy(oracle.bench_input(A.num_cols))
        # one gathered SpMV
        out_full = torch.empty(A.num_rows, dtype=torch.float64)
        D.spmv_gather(x0, out_full)
        lam, x = D.power_iteration(x0, iters)
        res = dict(rank=rank, bounds=D.bounds.tolist(), counts=D.counts, r0=sl.row_begin, r1=sl.row_end,
                   y1=out_full.numpy().copy(), lam=lam, x=x.numpy().copy(), interior=D.interior,
                   groups=D.engine.num_groups, exchange=D.exchange)
        torch.save(res, out / f"rank{rank}.pt")
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind,tpg,dcs,overlap,exchange", [
    ("stencil", 128, 1, True, "auto"), ("stencil8", 128, 32, True, "allgather"), ("stencil8", 128, 1, True, "halo"),
    ("powerlaw", 32, 4, True, "auto"), ("powerlaw", 32, 4, True, "halo"), ("stencil", 128, 1, False, "auto")])
def test_two_rank_power_iteration_gloo(tmp_path, kind, tpg, dcs, overlap, exchange):
    import oracle

    port = 29500 + (os.getpid() % 1000)
    iters = 12
    mp.start_processes(_worker, args=(2, port, kind, tpg, dcs, iters, tmp_path, overlap, exchange), nprocs=2,
                       join=True,
                       start_method="spawn")
    res = [torch.load(tmp_path / f"rank{r}.pt", weights_only=False) for r in range(2)]
    A = _matrix(kind)
    orc = oracle.orc()
    x0 = oracle.bench_input(A.num_cols)
    # split: nnz-balanced, contiguous, covering all rows
    b = res[0]["bounds"]
    if kind == "stencil8":
        assert res[0]["counts"][0] == res[0]["counts"][1]
    assert b[0] == 0 and b[-1] == A.num_rows and res[0]["r1"] == res[1]["r0"]
    half = int(A.row_pointers[-1]) // 2
    assert A.row_pointers[b[1] - 1] < half <= A.row_pointers[b[1]] or b[1] == np.searchsorted(A.row_pointers, half)
    # gathered first SpMV == full-matrix reference SpMV (per-row bound; bit-exact rows within each slice)
    y_full = orc.spmv_csr(A, x0)
    absrow = orc.abs_row_sums(A, x0)
    for r in res:
        assert np.all(np.abs(r["y1"] - y_full) <= 1e-12 * absrow)
        assert np.array_equal(r["y1"], res[0]["y1"])  # every rank holds the same gathered y
    if exchange == "halo" or (overlap and exchange == "auto" and kind.startswith("stencil")):
        assert all(r["exchange"] == "halo" for r in res)
    if not overlap or exchange == "allgather":
        assert all(r["exchange"] == "allgather" for r in res)
    if overlap and kind.startswith("stencil"):
        for r in res:  # a stencil slice: interior groups between its boundary layers (none at the matrix ends)
            ga, gb = r["interior"]
            assert ga < gb
            assert (ga > 0) == (r["r0"] > 0) and (gb < r["groups"]) == (r["r1"] < A.num_rows)
    lam_ref, x_ref = reference_power_iteration(A, x0, iters, tpg, dcs)
    for r in res:
        assert abs(r["lam"] - lam_ref) <= 1e-10 * abs(lam_ref)
        assert np.max(np.abs(r["x"] - x_ref)) <= 1e-9


def test_partition_bounds_match_c_abi(argcsr):
    from paper_1203_5737_b200.multigpu import partition_bounds

    rng = np.random.default_rng(0)
    for _ in range(50):
        n = int(rng.integers(1, 300))
        lens = rng.integers(0, 50, n)
        lens[rng.integers(0, n)] = 3000
        rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint64)
        for parts in (1, 2, 3, 4, 8):
            assert np.array_equal(partition_bounds(rp, parts), argcsr.partition_rows(rp, parts))
