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


@pytest.mark.parametrize("heavy", ["default", "ARGCSR_HEAVY_U=16", "ARGCSR_HEAVY_RUNS=1"])
def test_fused_scale_heavy_groups(argcsr, orc, heavy, monkeypatch):
    """The fused scale through the long-chunk kernel variants."""
    from helpers import powerlaw_csr

    if heavy != "default":
        monkeypatch.setenv(*heavy.split("="))
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
    import oracle
    from paper_1203_5737_b200.multigpu import DistributedArgCsr

    A = stencil27(20)
    D = DistributedArgCsr(A.num_rows, A.num_cols, A.row_pointers, A.columns, A.values, tpg, dcs,
                          device=torch.device("cuda", 0))
    x0 = oracle.bench_input(A.num_cols)
    lam, x = D.power_iteration(torch.from_numpy(x0).cuda(), 30)
    lam_ref, x_ref = reference_power_iteration(A, x0, 30, tpg, dcs)
    assert abs(lam - lam_ref) <= 1e-10 * abs(lam_ref)
    assert np.max(np.abs(x.cpu().numpy() - x_ref)) <= 1e-9


@pytest.mark.parametrize("x_remap", ["auto", "on"])
def test_interior_boundary_split_is_bit_identical(argcsr, x_remap):
    """The overlapped multi-GPU step computes interior groups, then the two
    boundary ranges (the last one reusing x'); together they equal one SpMV."""
    from paper_1203_5737_b200.multigpu import DeviceEngine, interior_group_range, slice_rows

    A = stencil27(18)
    sl = slice_rows(A.row_pointers, A.columns, A.values, A.num_cols, 0, A.num_rows)
    eng = DeviceEngine(sl, 128, 1, torch.device("cuda", 0))
    if x_remap == "on":
        eng.m = argcsr.argcsr_from_csr((A.num_rows, A.num_cols, A.row_pointers, A.columns, A.values), 128, 1,
                                       x_remap="on")
    r0, r1 = A.num_rows // 3, 2 * A.num_rows // 3  # pretend this rank owns the middle third of x
    ga, gb = interior_group_range(A.row_pointers, A.columns, eng.group_first_rows(), r0, r1)
    assert 0 < ga < gb < eng.num_groups
    x = torch.linspace(-2, 2, A.num_cols, dtype=torch.float64, device="cuda")
    s = torch.tensor([0.37], dtype=torch.float64, device="cuda")
    y_full = torch.empty(A.num_rows, dtype=torch.float64, device="cuda")
    eng.spmv(x, y_full, s)
    y = torch.full_like(y_full, float("nan"))
    eng.spmv_range(x, y, ga, gb, s)
    eng.spmv_range(x, y, 0, ga, s)
    eng.spmv_range(x, y, gb, eng.num_groups, s, reuse_x=True)
    assert bits(y.cpu().numpy()) == bits(y_full.cpu().numpy())


@pytest.mark.parametrize("exchange", ["auto", "p2p"])
def test_power_iteration_engine_on_side_stream(exchange):
    """The engine converted under a side stream (as bench.py sets it up), the
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
