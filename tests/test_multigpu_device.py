"""The multi-GPU layer on the device path (world size 1 on one B200): the
fused normalisation of argcsr_dev_spmv_scaled is bit-identical to scaling x
first, and the power iteration matches the single-process CPU run."""
import numpy as np
import pytest
import torch

from helpers import bits, stencil27
from test_multigpu_gloo import reference_power_iteration

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("x_remap", ["auto", "on"])
def test_fused_scale_is_bit_identical(argcsr, orc, x_remap):
    A = stencil27(16)
    m = argcsr.argcsr_from_csr((A.num_rows, A.num_cols, A.row_pointers, A.columns, A.values), 128, 1,
                               x_remap=x_remap)
    assert m.x_remap == (x_remap == "on")
    x = torch.linspace(-3, 3, A.num_cols, dtype=torch.float64, device="cuda")
    s = torch.tensor([1.0 / 7.3], dtype=torch.float64, device="cuda")
    y1 = torch.empty(A.num_rows, dtype=torch.float64, device="cuda")
    m.spmv_scaled_device(x.data_ptr(), s.data_ptr(), y1.data_ptr(), torch.cuda.current_stream().cuda_stream)
    y2 = argcsr.spmv_torch(m, x * s)
    assert bits(y1.cpu().numpy()) == bits(y2.cpu().numpy())
    ref = orc.spmv_argcsr(orc.argcsr_from_csr(A, 128, 1), (x * s).cpu().numpy())
    assert bits(y1.cpu().numpy()) == bits(ref)


@pytest.mark.parametrize("heavy", ["default", "ARGCSR_HEAVY_PIPE=1", "ARGCSR_HEAVY_PIPE=0"])
def test_fused_scale_heavy_groups(argcsr, orc, heavy, monkeypatch):
    """The fused scale through the long-chunk kernel variants."""
    from helpers import powerlaw_csr

    if heavy != "default":
        for kv in heavy.split(","):
            monkeypatch.setenv(*kv.split("="))
        argcsr._ext.reload_options()
    A = powerlaw_csr(20000, 20000, seed=5, heavy_rows=[(3, 12000), (9000, 7000)])
    m = argcsr.argcsr_from_csr((A.num_rows, A.num_cols, A.row_pointers, A.columns, A.values), 128, 1)
    assert m.heavy_groups > 0
    x = torch.linspace(-3, 3, A.num_cols, dtype=torch.float64, device="cuda")
    s = torch.tensor([1.0 / 7.3], dtype=torch.float64, device="cuda")
    y1 = torch.empty(A.num_rows, dtype=torch.float64, device="cuda")
    m.spmv_scaled_device(x.data_ptr(), s.data_ptr(), y1.data_ptr(), torch.cuda.current_stream().cuda_stream)
    ref = orc.spmv_argcsr(orc.argcsr_from_csr(A, 128, 1), (x * s).cpu().numpy())
    assert bits(y1.cpu().numpy()) == bits(ref)


@pytest.mark.parametrize("tpg,dcs", [(128, 1), (128, 32)])
def test_power_iteration_single_rank(tpg, dcs):
    """DistributedArgCsr (the C-ABI argcsr_mgpu_*) at world size 1."""
    import oracle
    from paper_1203_5737_b200.multigpu import DistributedArgCsr

    A = stencil27(20)
    D = DistributedArgCsr(A.num_rows, A.num_cols, A.row_pointers, A.columns, A.values, tpg, dcs,
                          device=torch.device("cuda", 0))
    assert D.exchange == "none" and (D.r0, D.r1) == (0, A.num_rows)
    x0 = oracle.bench_input(A.num_cols)
    lam, x = D.power_iteration(torch.from_numpy(x0).cuda(), 30)
    lam_ref, x_ref = reference_power_iteration(A, x0, 30, tpg, dcs)
    assert abs(lam - lam_ref) <= 1e-10 * abs(lam_ref)
    assert np.max(np.abs(x.cpu().numpy() - x_ref)) <= 1e-9
    # a second run on the same handle gives the same bits (deterministic norms)
    lam2, x2 = D.power_iteration(torch.from_numpy(x0).cuda(), 30)
    assert lam2 == lam and torch.equal(x2, x)
    D.close()


@pytest.mark.parametrize("kind", ["stencil", "powerlaw"])
def test_power_iteration_one_rank_nccl(argcsr, kind):
    """A one-rank NCCL communicator (argcsr_mgpu_create_rank with an
    ncclUniqueId): the all-reduce of ||y||^2 and the in-place all-gather run
    through NCCL every step; the result matches the CPU run and the
    communicator reports no asynchronous error."""
    import oracle
    from helpers import powerlaw_csr

    A = stencil27(18) if kind == "stencil" else powerlaw_csr(8000, 8000, seed=3, heavy_rows=[(5, 5000)])
    rp = torch.from_numpy(A.row_pointers.astype(np.int64))
    cols = torch.from_numpy(A.columns)
    vals = torch.from_numpy(A.values)
    h = argcsr._ext.MultiGpu.create_rank(A.num_rows, A.num_cols, A.nnz, rp.data_ptr(), cols.data_ptr(),
                                         vals.data_ptr(), "float64", False, 0, 1, argcsr._ext.mgpu_unique_id(),
                                         128, 1, 0, 0, 0)
    x0 = oracle.bench_input(A.num_cols)
    xh = x0.copy()
    lam = h.power_iteration(25, xh)
    h.check()
    lam_ref, x_ref = reference_power_iteration(A, x0, 25, 128, 1)
    assert abs(lam - lam_ref) <= 1e-10 * abs(lam_ref)
    assert np.max(np.abs(xh - x_ref)) <= 1e-9
    # iterated SpMV through the same handle (spmv_gather: SpMV + all-gather)
    x = torch.from_numpy(x0).cuda()
    out = torch.empty_like(x)
    h.spmv_gather([x.data_ptr()], [out.data_ptr()], [torch.cuda.current_stream().cuda_stream])
    ref = oracle.orc().spmv_argcsr(oracle.orc().argcsr_from_csr(A, 128, 1), x0)
    assert bits(out.cpu().numpy()) == bits(ref)
    h.free()


def test_spmv_norm2_fused_and_deterministic(argcsr, orc):
    """argcsr_dev_spmv_norm2: y bit-identical to the plain SpMV, ||y||^2 from
    the epilogue partials equal (to rounding) to the sum of squares, and the
    same bits on every call; the norm2 scale mode equals scaling by
    1/sqrt(s2) first."""
    from helpers import powerlaw_csr

    for A in (stencil27(20), powerlaw_csr(30000, 30000, seed=5, heavy_rows=[(3, 12000)])):
        m = argcsr.argcsr_from_csr((A.num_rows, A.num_cols, A.row_pointers, A.columns, A.values), 128, 1)
        x = torch.linspace(-2, 2, A.num_cols, dtype=torch.float64, device="cuda")
        y = torch.empty(A.num_rows, dtype=torch.float64, device="cuda")
        n2 = torch.zeros(1, dtype=torch.float64, device="cuda")
        st = torch.cuda.current_stream().cuda_stream
        m.spmv_norm2_device(x.data_ptr(), 0, y.data_ptr(), n2.data_ptr(), False, st)
        ref = orc.spmv_argcsr(orc.argcsr_from_csr(A, 128, 1), x.cpu().numpy())
        assert bits(y.cpu().numpy()) == bits(ref)
        want = float(np.dot(ref, ref))
        assert abs(float(n2.item()) - want) <= 1e-12 * want
        first = float(n2.item())
        for _ in range(3):
            m.spmv_norm2_device(x.data_ptr(), 0, y.data_ptr(), n2.data_ptr(), False, st)
            assert float(n2.item()) == first
        s2 = torch.tensor([7.25], dtype=torch.float64, device="cuda")
        m.spmv_norm2_device(x.data_ptr(), s2.data_ptr(), y.data_ptr(), n2.data_ptr(), True, st)
        xs = (x * (1.0 / torch.sqrt(s2))).cpu().numpy()
        assert bits(y.cpu().numpy()) == bits(orc.spmv_argcsr(orc.argcsr_from_csr(A, 128, 1), xs))


@pytest.mark.parametrize("x_remap", ["auto", "on"])
def test_interior_boundary_split_is_bit_identical(argcsr, x_remap):
    """The overlapped multi-GPU step computes interior groups, then the two
    boundary ranges (the last one reusing x'); together they equal one SpMV."""
    from paper_1203_5737_b200.multigpu import interior_group_range

    A = stencil27(18)
    m = argcsr.argcsr_from_csr((A.num_rows, A.num_cols, A.row_pointers, A.columns, A.values), 128, 1,
                               x_remap=x_remap)
    gf = np.concatenate([m.groups_array[:, 0], [A.num_rows]]).astype(np.uint64)
    r0, r1 = A.num_rows // 3, 2 * A.num_rows // 3  # pretend this rank owns the middle third of x
    ga, gb = interior_group_range(A.row_pointers, A.columns, gf, r0, r1)
    assert 0 < ga < gb < m.num_groups
    x = torch.linspace(-2, 2, A.num_cols, dtype=torch.float64, device="cuda")
    s = torch.tensor([0.37], dtype=torch.float64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    y_full = torch.empty(A.num_rows, dtype=torch.float64, device="cuda")
    m.spmv_scaled_device(x.data_ptr(), s.data_ptr(), y_full.data_ptr(), st)
    y = torch.full_like(y_full, float("nan"))
    m.spmv_ex_device(x.data_ptr(), s.data_ptr(), ga, gb, y.data_ptr(), 0, st)
    m.spmv_ex_device(x.data_ptr(), s.data_ptr(), 0, ga, y.data_ptr(), 0, st)
    m.spmv_ex_device(x.data_ptr(), s.data_ptr(), gb, m.num_groups, y.data_ptr(), 1, st)
    assert bits(y.cpu().numpy()) == bits(y_full.cpu().numpy())


@pytest.mark.parametrize("exchange", ["auto", "p2p"])
def test_power_iteration_engine_on_side_stream(exchange):
    """The handle built under a side stream (as bench.py sets it up), the
    steps run on the caller's current stream: every product, norm and flag is
    ordered on the stream current at call time (a 262 k-row stencil is large
    enough for a cross-stream race to show)."""
    import oracle
    from paper_1203_5737_b200.multigpu import DistributedArgCsr

    A = stencil27(64)
    dev = torch.device("cuda", 0)
    side = torch.cuda.Stream(dev)
    with torch.cuda.stream(side):
        D = DistributedArgCsr(A.num_rows, A.num_cols, A.row_pointers, A.columns, A.values, 128, 1, device=dev,
                              exchange=exchange)
    x0 = oracle.bench_input(A.num_cols)
    lam, x = D.power_iteration(torch.from_numpy(x0).cuda(), 20)
    D.close()
    lam_ref, x_ref = reference_power_iteration(A, x0, 20, 128, 1)
    assert abs(lam - lam_ref) <= 1e-10 * abs(lam_ref)
    assert np.max(np.abs(x.cpu().numpy() - x_ref)) <= 1e-9


def test_cpp_mgpu_example_runs_on_the_device(tmp_path):
    """A C++ program drives the multi-GPU C-ABI: a one-rank NCCL job and three
    p2p virtual ranks, both checked against a CPU power iteration."""
    import subprocess
    from pathlib import Path

    root = Path(__file__).resolve().parent.parent
    exe = tmp_path / "mgpu_example"
    subprocess.run(["g++", "-std=c++20", "-O2", "-I", str(root / "include"), str(root / "examples" / "mgpu_example.cpp"),
                    "-L", str(root / "paper_1203_5737_b200"), "-largcsr_gpu",
                    f"-Wl,-rpath,{root / 'paper_1203_5737_b200'}", "-o", str(exe)], check=True)
    r = subprocess.run([str(exe), "20", "25"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count("ok=1") == 2
