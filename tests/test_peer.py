"""The fused multi-GPU step over peer memory (csrc/mgpu.cu, exchange p2p).

Only one GPU is available, so the protocol runs (a) as P virtual ranks of ONE
process sharing the device (argcsr_mgpu_create with the device listed P
times) -- each rank's SpMV epilogue stores its y slice into the other ranks'
x buffers, flags and partial norms travel the same way -- and (b) as two
processes sharing the GPU through real CUDA IPC handles (exchanged over the
gloo backend, argcsr_mgpu_p2p_export / _connect), the code path an 8-GPU box
runs over NVLink."""
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


def _virtual(argcsr, A, P, tpg=128, dcs=1):
    rp = torch.from_numpy(A.row_pointers.astype(np.int64))
    cols = torch.from_numpy(A.columns)
    vals = torch.from_numpy(A.values)
    return argcsr._ext.MultiGpu.create(A.num_rows, A.num_cols, A.nnz, rp.data_ptr(), cols.data_ptr(), vals.data_ptr(),
                                       "float64", False, [0] * P, tpg, dcs, 3)


@pytest.mark.parametrize("kind", ["stencil", "powerlaw"])
def test_spmv_peer_stores_bit_identical(argcsr, orc, kind):
    """argcsr_dev_spmv_peer: y and every peer target hold the oracle's bits
    (light tiles and heavy groups), other rows of the targets untouched."""
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


@pytest.mark.parametrize("P", [2, 3, 4])
@pytest.mark.parametrize("kind", ["stencil", "powerlaw"])
def test_peer_power_iteration_virtual_ranks(argcsr, kind, P):
    """Halo-only peer stores each step (the rows each peer's columns read),
    every row on the last step so every rank ends with all of x."""
    import oracle

    A = stencil27(16) if kind == "stencil" else powerlaw_csr(6000, 6000, seed=4, heavy_rows=[(7, 4000)])
    h = _virtual(argcsr, A, P)
    info = h.info()
    assert info["exchange"] == 3 and info["nranks"] == P and info["nlocal"] == P
    x0 = oracle.bench_input(A.num_cols)
    dev = [torch.from_numpy(x0).cuda() for _ in range(P)]
    outs = [torch.empty_like(dev[0]) for _ in range(P)]
    st = [torch.cuda.current_stream().cuda_stream] * P
    iters = 25
    h.begin([d.data_ptr() for d in dev], True, st)
    for i in range(iters):
        h.step(i == iters - 1, st)
    lam = h.finish([o.data_ptr() for o in outs], st)
    lam_ref, x_ref = reference_power_iteration(A, x0, iters, 128, 1)
    assert abs(lam - lam_ref) <= 1e-10 * abs(lam_ref)
    xs = [o.cpu().numpy() for o in outs]
    for x in xs:
        assert np.max(np.abs(x - x_ref)) <= 1e-9
    for x in xs[1:]:  # every rank assembled the same x, bit for bit
        assert bits(x) == bits(xs[0])
    # a second run on the same buffers (absolute step numbers: no stale flag passes)
    h.begin([d.data_ptr() for d in dev], True, st)
    for i in range(iters):
        h.step(i == iters - 1, st)
    assert h.finish([o.data_ptr() for o in outs], st) == lam
    h.free()


@pytest.mark.parametrize("P", [2, 3])
def test_peer_iterated_spmv_virtual_ranks(argcsr, orc, P):
    """normalize=False: x_{k+1} = A x_k assembled on every rank; each slice is
    the oracle's SpMV of that rank's slice conversion, bit for bit."""
    import oracle
    from paper_1203_5737_b200.multigpu import partition_bounds

    A = powerlaw_csr(5000, 5000, seed=8, heavy_rows=[(9, 3000)])
    A.values[:] = A.values / np.abs(A.values).sum() * 50  # keep x bounded over the steps
    h = _virtual(argcsr, A, P)
    b = partition_bounds(A.row_pointers, P)
    x0 = np.linspace(-1, 1, A.num_cols)
    dev = [torch.from_numpy(x0).cuda() for _ in range(P)]
    outs = [torch.empty_like(dev[0]) for _ in range(P)]
    st = [torch.cuda.current_stream().cuda_stream] * P
    h.begin([d.data_ptr() for d in dev], False, st)
    for i in range(4):
        h.step(i == 3, st)
    h.finish([o.data_ptr() for o in outs], st)
    refs = []
    for p in range(P):
        r0, r1 = int(b[p]), int(b[p + 1])
        a, e = int(A.row_pointers[r0]), int(A.row_pointers[r1])
        sl = oracle.Csr(r1 - r0, A.num_cols, (A.row_pointers[r0:r1 + 1] - A.row_pointers[r0]).astype(np.uint64),
                        A.columns[a:e], A.values[a:e])
        refs.append(orc.argcsr_from_csr(sl, 128, 1))
    x = x0.copy()
    for _ in range(4):
        x = np.concatenate([orc.spmv_argcsr(M, x) for M in refs])
    for o in outs:
        assert bits(o.cpu().numpy()) == bits(x)
    h.free()


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
        # NCCL refuses two ranks on one GPU: the IPC handles go over gloo instead
        D = DistributedArgCsr(A.num_rows, A.num_cols, A.row_pointers, A.columns, A.values, 128, 1,
                              device=torch.device("cuda", 0), exchange="p2p", nccl=False)
        assert D.exchange == "p2p"
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
