"""The multi-GPU layer's host logic on CPU, world size 2 with
the gloo backend.  The layer itself is C++ behind the C-ABI (csrc/mgpu.cu);
its host planning entry points run without a device:

* argcsr_partition_rows       nnz-balanced contiguous slices;
* argcsr_plan_interior        the groups whose rows read only the slice's own
                              x rows (computed under the exchange);
* argcsr_plan_needed          the rows of every other slice a slice reads (the
                              halo plan: what each rank receives / sends).

The two-rank test drives those plans exactly as argcsr_mgpu_create_rank does
-- the receive lists are exchanged between the ranks (here over gloo, on the
box over NCCL) to become the send lists -- and runs the halo-exchange power
iteration with the test-only oracle standing in for each rank's GPU, against
a single-process CPU run.  The device path itself is covered by
tests/test_multigpu_device.py and tests/test_peer.py."""
import os
import sys
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parent.parent


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
        return stencil27(9)  # 729 rows: uneven split
    if kind == "stencil8":
        return stencil27(8)  # 512 rows: even split
    return powerlaw_csr(3001, 3001, seed=4, heavy_rows=[(7, 2000)])


def _slice(A, r0, r1):
    import oracle

    a, b = int(A.row_pointers[r0]), int(A.row_pointers[r1])
    return oracle.Csr(r1 - r0, A.num_cols, (A.row_pointers[r0:r1 + 1] - A.row_pointers[r0]).astype(np.uint64),
                      A.columns[a:b], A.values[a:b])


def _worker(rank, world, port, kind, tpg, dcs, iters, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, str(ROOT))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import paper_1203_5737_b200 as argcsr
        from paper_1203_5737_b200.multigpu import interior_group_range, needed_rows, partition_bounds

        orc = oracle.orc()
        A = _matrix(kind)
        b = partition_bounds(A.row_pointers, world)
        assert np.array_equal(b, argcsr.partition_rows(A.row_pointers, world))
        r0, r1 = int(b[rank]), int(b[rank + 1])
        S = _slice(A, r0, r1)
        M = orc.argcsr_from_csr(S, tpg, dcs)  # the slice's conversion (the GPU's is checked bit-exact elsewhere)
        gfirst = np.concatenate([M.groups[:, 0], [S.num_rows]]).astype(np.uint64)
        ga, gb = interior_group_range(S.row_pointers, S.columns, gfirst, r0, r1)
        # halo plan: rows I read from every owner; the owners learn them (all-to-all of the lists)
        need = needed_rows(S.columns, A.num_cols, b, rank)
        sends = [None] * world
        dist.all_gather_object(sends, [n.tolist() for n in need])
        send_to = {q: sends[q][rank] for q in range(world) if q != rank}  # rows q reads from me
        # power iteration with the halo exchange over gloo
        x = oracle.bench_input(A.num_cols)
        scale, s2 = 1.0, 0.0
        for _ in range(iters):
            y = orc.spmv_argcsr(M, x * scale)
            part = torch.tensor([float(np.dot(y, y))], dtype=torch.float64)
            dist.all_reduce(part)
            s2 = float(part.item())
            x = x.copy()
            x[r0:r1] = y
            for q in range(world):  # exchange: send my rows q reads, receive the rows I read from q
                if q == rank:
                    continue
                out_t = torch.from_numpy(np.ascontiguousarray(x[np.asarray(send_to[q], np.int64)]))
                in_t = torch.empty(len(need[q]), dtype=torch.float64)
                if rank < q:
                    dist.send(out_t, q)
                    dist.recv(in_t, q)
                else:
                    dist.recv(in_t, q)
                    dist.send(out_t, q)
                x[np.asarray(need[q], np.int64)] = in_t.numpy()
            scale = 1.0 / np.sqrt(s2)
        # assemble (the last step of the device run exchanges every row)
        full = [None] * world
        dist.all_gather_object(full, x[r0:r1].copy())
        x = np.concatenate(full) * scale
        res = dict(rank=rank, bounds=b.tolist(), r0=r0, r1=r1, lam=float(np.sqrt(s2)), x=x, interior=(ga, gb),
                   groups=int(M.groups.shape[0]), need=[len(n) for n in need])
        torch.save(res, out / f"rank{rank}.pt")
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind,tpg,dcs", [("stencil", 128, 1), ("stencil8", 128, 32), ("powerlaw", 32, 4)])
def test_two_rank_halo_power_iteration_gloo(tmp_path, kind, tpg, dcs):
    import oracle

    port = 29500 + (os.getpid() % 1000)
    iters = 12
    mp.start_processes(_worker, args=(2, port, kind, tpg, dcs, iters, tmp_path), nprocs=2, join=True,
                       start_method="spawn")
    res = [torch.load(tmp_path / f"rank{r}.pt", weights_only=False) for r in range(2)]
    A = _matrix(kind)
    b = res[0]["bounds"]
    assert b[0] == 0 and b[-1] == A.num_rows and res[0]["r1"] == res[1]["r0"]
    half = int(A.row_pointers[-1]) // 2
    assert b[1] == np.searchsorted(A.row_pointers, half)
    if kind.startswith("stencil"):
        n = 9 if kind == "stencil" else 8
        for r in res:  # a stencil slice: interior groups between its boundary layers; a plane of halo
            ga, gb = r["interior"]
            assert ga < gb
            assert (ga > 0) == (r["r0"] > 0) and (gb < r["groups"]) == (r["r1"] < A.num_rows)
            assert 0 < sum(r["need"]) <= n * n + n + 1
    lam_ref, x_ref = reference_power_iteration(A, oracle.bench_input(A.num_cols), iters, tpg, dcs)
    for r in res:
        assert abs(r["lam"] - lam_ref) <= 1e-10 * abs(lam_ref)
        assert np.max(np.abs(r["x"] - x_ref)) <= 1e-9


def test_plan_needed_matches_numpy(argcsr):
    from helpers import powerlaw_csr, stencil27
    from paper_1203_5737_b200.multigpu import needed_rows, partition_bounds

    for A in (stencil27(10), powerlaw_csr(2000, 2500, seed=3, heavy_rows=[(5, 1500)])):
        for P in (1, 2, 3, 5):
            b = partition_bounds(A.row_pointers, P)
            for p in range(P):
                S = _slice(A, int(b[p]), int(b[p + 1]))
                got = needed_rows(S.columns, A.num_cols, b, p)
                c = np.unique(S.columns.astype(np.int64))
                for q in range(P):
                    want = c[(c >= b[q]) & (c < b[q + 1])] if q != p else np.zeros(0, np.int64)
                    assert np.array_equal(got[q], want.astype(np.uint64))


def test_plan_interior_matches_numpy(argcsr):
    from helpers import powerlaw_csr, stencil27
    from paper_1203_5737_b200.multigpu import interior_group_range

    import oracle

    orc = oracle.orc()
    for A in (stencil27(12), powerlaw_csr(3000, 3000, seed=6)):
        M = orc.argcsr_from_csr(A, 128, 1)
        gf = np.concatenate([M.groups[:, 0], [A.num_rows]]).astype(np.uint64)
        for r0, r1 in ((0, A.num_rows), (A.num_rows // 3, 2 * A.num_rows // 3), (0, 10)):
            ga, gb = interior_group_range(A.row_pointers, A.columns, gf, r0, r1)
            row = np.repeat(np.arange(A.num_rows), np.diff(A.row_pointers.astype(np.int64)))
            bad_rows = np.zeros(A.num_rows, bool)
            bad_rows[row[(A.columns < r0) | (A.columns >= r1)]] = True
            good = np.array([not bad_rows[gf[g]:gf[g + 1]].any() for g in range(len(gf) - 1)] + [False])
            best, run = (0, 0), None
            for g, ok in enumerate(good):
                if ok and run is None:
                    run = g
                if not ok and run is not None:
                    if g - run > best[1] - best[0]:
                        best = (run, g)
                    run = None
            assert (ga, gb) == best


def test_partition_rule(argcsr):
    """argcsr_partition_rows: lower_bound(rp, p * nnz / P), parts kept non-empty."""
    from paper_1203_5737_b200.multigpu import partition_bounds

    rng = np.random.default_rng(0)
    for _ in range(50):
        n = int(rng.integers(1, 300))
        lens = rng.integers(0, 50, n)
        lens[rng.integers(0, n)] = 3000
        rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint64)
        nnz = int(rp[-1])
        for parts in (1, 2, 3, 4, 8):
            b = partition_bounds(rp, parts)
            assert b[0] == 0 and b[-1] == n and np.all(np.diff(b.astype(np.int64)) >= (1 if n >= parts else 0))
            for p in range(1, parts):
                want = int(np.searchsorted(rp, nnz * p // parts, side="left"))
                lo = int(b[p - 1]) + (1 if n >= parts else 0)
                hi = n - (parts - p) if n >= parts else n
                assert int(b[p]) == min(max(want, lo), hi)


def test_wrapper_fails_loudly_without_a_device(argcsr):
    """DistributedArgCsr is the C-ABI: no device -> CudaError, no CPU fallback."""
    if torch.cuda.is_available():
        pytest.skip("a device is present")
    from helpers import stencil27
    from paper_1203_5737_b200.multigpu import DistributedArgCsr

    A = stencil27(6)
    with pytest.raises(argcsr.CudaError):
        DistributedArgCsr(A.num_rows, A.num_cols, A.row_pointers, A.columns, A.values, device=torch.device("cpu"))
