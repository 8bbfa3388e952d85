"""The fused multi-GPU step over peer memory (paper_1203_5737_b200/peer.py).

Only one GPU is available, so the protocol runs (a) as P virtual ranks on one
device -- each rank's SpMV epilogue stores its y slice into the other ranks'
x buffers, flags and partial norms travel the same way -- and (b) as two
processes sharing the GPU through real CUDA IPC handles (exchanged with the
gloo backend), the code path an 8-GPU box runs over NVLink."""
import os
import sys
import traceback
from pathlib import Path

import numpy as np
import pytest
import torch

from helpers import bits, powerlaw_csr, stencil27
from test_multigpu_gloo import reference_power_iteration

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def _engines(A, P, tpg=128, dcs=1):
    from paper_1203_5737_b200.multigpu import DeviceEngine, partition_bounds, slice_rows

    b = partition_bounds(A.row_pointers, P)
    dev = torch.device("cuda", 0)
    engs = [DeviceEngine(slice_rows(A.row_pointers, A.columns, A.values, A.num_cols, int(b[p]), int(b[p + 1])),
                         tpg, dcs, dev) for p in range(P)]
    return b, engs


@pytest.mark.parametrize("kind", ["stencil", "powerlaw"])
def test_spmv_peer_stores_bit_identical(argcsr, orc, kind):
    """argcsr_dev_spmv_peer: y and every peer target hold the oracle's bits
    (light tiles and heavy groups), other rows of the targets untouched."""
    import oracle

    A = stencil27(14) if kind == "stencil" else powerlaw_csr(30000, 30000, seed=9, heavy_rows=[(11, 15000)])
    m = argcsr.argcsr_from_csr((A.num_rows, A.num_cols, A.row_pointers, A.columns, A.values), 128, 1)
    x = torch.linspace(-2, 3, A.num_cols, dtype=torch.float64, device="cuda")
    s = torch.tensor([0.75], dtype=torch.float64, device="cuda")
    y = torch.empty(A.num_rows, dtype=torch.float64, device="cuda")
    r0 = 5
    targets = [torch.full((A.num_rows + 10,), 3.5, dtype=torch.float64, device="cuda") for _ in range(3)]
    m.spmv_peer_device(x.data_ptr(), s.data_ptr(), 0, m.num_groups, y.data_ptr(),
                       [t.data_ptr() + r0 * 8 for t in targets], stream=torch.cuda.current_stream().cuda_stream)
    ref = orc.spmv_argcsr(orc.argcsr_from_csr(A, 128, 1), (x * s).cpu().numpy())
    assert bits(y.cpu().numpy()) == bits(ref)
    for t in targets:
        t = t.cpu().numpy()
        assert bits(t[r0:r0 + A.num_rows]) == bits(ref)
        assert np.all(t[:r0] == 3.5) and np.all(t[r0 + A.num_rows:] == 3.5)
    with pytest.raises(argcsr.ParameterError):
        m.spmv_peer_device(x.data_ptr(), 0, 0, m.num_groups, y.data_ptr(), [t.data_ptr() for t in targets * 3])
    # row ranges: peer 0 gets rows [100, 300), peer 1 none, peer 2 all
    for t in targets:
        t.fill_(3.5)
    m.spmv_peer_device(x.data_ptr(), s.data_ptr(), 0, m.num_groups, y.data_ptr(),
                       [t.data_ptr() + r0 * 8 for t in targets], peer_rows=[100, 300, 0, 0, 0, A.num_rows],
                       stream=torch.cuda.current_stream().cuda_stream)
    t0, t1, t2 = (t.cpu().numpy()[r0:r0 + A.num_rows] for t in targets)
    assert bits(t0[100:300]) == bits(ref[100:300]) and np.all(t0[:100] == 3.5) and np.all(t0[300:] == 3.5)
    assert np.all(t1 == 3.5)
    assert bits(t2) == bits(ref)


@pytest.mark.parametrize("halo", [False, True])
@pytest.mark.parametrize("P", [1, 2, 3, 4])
@pytest.mark.parametrize("kind", ["stencil", "powerlaw"])
def test_peer_power_iteration_virtual_ranks(kind, P, halo):
    """Full stores, or halo-only stores (each peer gets the rows its columns
    read; the last step stores everything so every rank ends with all of x)."""
    import oracle
    from paper_1203_5737_b200.multigpu import slice_rows
    from paper_1203_5737_b200.peer import power_iteration_local

    A = stencil27(16) if kind == "stencil" else powerlaw_csr(6000, 6000, seed=4, heavy_rows=[(7, 4000)])
    b, engs = _engines(A, P)
    cols = [slice_rows(A.row_pointers, A.columns, A.values, A.num_cols, int(b[p]), int(b[p + 1])).columns
            for p in range(P)] if halo else None
    x0 = oracle.bench_input(A.num_cols)
    out = power_iteration_local(engs, b, A.num_cols, torch.from_numpy(x0).cuda(), 25, slice_columns=cols)
    lam_ref, x_ref = reference_power_iteration(A, x0, 25, 128, 1)
    xs = [x.cpu().numpy() for _, x in out]
    for lam, x in zip((o[0] for o in out), xs):
        assert abs(lam - lam_ref) <= 1e-10 * abs(lam_ref)
        assert np.max(np.abs(x - x_ref)) <= 1e-9
    for x in xs[1:]:  # every rank assembled the same x, bit for bit
        assert bits(x) == bits(xs[0])


@pytest.mark.parametrize("P", [2, 3])
def test_peer_iterated_spmv_virtual_ranks(orc, P):
    """normalize=False: x_{k+1} = A x_k assembled on every rank; each step's
    slices are the oracle's SpMV of that rank's slice conversion, bit for bit."""
    from paper_1203_5737_b200.multigpu import slice_rows
    from paper_1203_5737_b200.peer import power_iteration_local
    import oracle

    A = powerlaw_csr(5000, 5000, seed=8, heavy_rows=[(9, 3000)])
    A.values[:] = A.values / np.abs(A.values).sum() * 50  # keep x bounded over the steps
    b, engs = _engines(A, P)
    x0 = np.linspace(-1, 1, A.num_cols)
    out = power_iteration_local(engs, b, A.num_cols, torch.from_numpy(x0).cuda(), 4, normalize=False)
    x = x0.copy()
    refs = []
    for p in range(P):
        sl = slice_rows(A.row_pointers, A.columns, A.values, A.num_cols, int(b[p]), int(b[p + 1]))
        refs.append(orc.argcsr_from_csr(oracle.Csr(sl.num_rows, A.num_cols, np.asarray(sl.row_pointers, np.uint64),
                                                   np.asarray(sl.columns, np.int32), np.asarray(sl.values)), 128, 1))
    for _ in range(4):
        x = np.concatenate([orc.spmv_argcsr(M, x) for M in refs])
    for xr in out:
        assert bits(xr.cpu().numpy()) == bits(x)


def _ipc_worker(rank, world, port, kind, out_dir):
    try:
        sys.path.insert(0, str(ROOT))
        sys.path.insert(0, str(ROOT / "tests"))
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        import torch.distributed as dist

        import oracle
        from paper_1203_5737_b200.multigpu import DistributedArgCsr

        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        A = stencil27(12) if kind == "stencil" else powerlaw_csr(5000, 5000, seed=2, heavy_rows=[(3, 3000)])
        D = DistributedArgCsr(A.num_rows, A.num_cols, A.row_pointers, A.columns, A.values, 128, 1,
                              device=torch.device("cuda", 0), exchange="p2p")
        assert D.exchange == "p2p" and D.peer.peers == [1 - rank]
        x0 = oracle.bench_input(A.num_cols)
        lam, x = D.power_iteration(torch.from_numpy(x0).cuda(), 12)
        lam2, x2 = D.power_iteration(torch.from_numpy(x0).cuda(), 12)  # a second run on the same buffers
        assert lam2 == lam and torch.equal(x2, x)
        np.save(os.path.join(out_dir, f"x{rank}.npy"), x.cpu().numpy())
        np.save(os.path.join(out_dir, f"lam{rank}.npy"), np.array([lam]))
        D.close()
        dist.destroy_process_group()
    except Exception:
        with open(os.path.join(out_dir, f"err{rank}.txt"), "w") as f:
            f.write(traceback.format_exc())
        raise


@pytest.mark.timeout(600)
@pytest.mark.parametrize("kind", ["stencil", "powerlaw"])
def test_peer_power_iteration_two_processes_ipc(kind, tmp_path):
    """Two processes on one GPU: CUDA IPC buffers, flags and peer stores
    across process boundaries (the multi-process code path)."""
    import socket

    import oracle
    import torch.multiprocessing as mp

    with socket.socket() as s_:
        s_.bind(("127.0.0.1", 0))
        port = s_.getsockname()[1]
    mp.start_processes(_ipc_worker, args=(2, port, kind, str(tmp_path)), nprocs=2, join=True, start_method="spawn")
    A = stencil27(12) if kind == "stencil" else powerlaw_csr(5000, 5000, seed=2, heavy_rows=[(3, 3000)])
    lam_ref, x_ref = reference_power_iteration(A, oracle.bench_input(A.num_cols), 12, 128, 1)
    xs = [np.load(tmp_path / f"x{r}.npy") for r in range(2)]
    for r in range(2):
        lam = float(np.load(tmp_path / f"lam{r}.npy")[0])
        assert abs(lam - lam_ref) <= 1e-10 * abs(lam_ref)
        assert np.max(np.abs(xs[r] - x_ref)) <= 1e-9
    assert bits(xs[0]) == bits(xs[1])
