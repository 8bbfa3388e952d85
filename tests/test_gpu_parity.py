"""Parity of the CUDA path (through the C-ABI) with the CPU oracle.

Mirrors the reference's known-answer suite proj/tests/test_argcsr.cpp and the
acceptance criteria proj/tests/acceptance.cpp:76-198 on the device:
conversion is compared byte-for-byte (groups, threads_mapping, values,
columns) and fp64 SpMV bit-for-bit against the oracle's spmv_argcsr (same
summation order, no FMA).  The tolerance bound of the north_star,
|y_gpu - y_ref| <= 1e-12 * sum_j |a_ij x_j| per row (fp64) / 1e-5 (fp32), is
checked against the oracle's CSR product as well.
"""
import numpy as np
import pytest

from helpers import LAYOUTS, assert_same_layout, bits, np_corpus, powerlaw_csr, stencil27, to_dev
from oracle import Csr

pytestmark = pytest.mark.gpu

FP64_TOL = 1e-12
FP32_TOL = 1e-5


def e8(argcsr):
    return argcsr.csr_from_triplets(8, 8, [(r, r, 1.0) for r in range(7)] + [(7, c, 1.0) for c in range(8)])


def within_bound(y, y_ref, absrow, tol):
    return np.all(np.abs(np.asarray(y, np.float64) - y_ref) <= tol * absrow)


# ---------------------------------------------------------------- known answers
def test_e8_anatomy_chunk_budget_2(argcsr):  # test_argcsr.cpp:91-110
    m = argcsr.argcsr_from_csr(e8(argcsr), 12, 2)
    assert m.num_groups == 1
    assert m.groups[0] == argcsr.GroupInfo(0, 8, 0, 2)
    assert list(m.threads_mapping) == [1, 2, 3, 4, 5, 6, 7, 11]
    assert m.total_slots == 24
    assert argcsr.chunk_entries(m, 0, 7) == [(1.0, 0), (1.0, 1)]
    assert m.columns[0 * 12 + 0] == 0
    assert m.columns[1 * 12 + 0] == argcsr.kPaddingColumn
    assert argcsr.chunk_entries(m, 0, 11) == []


def test_e8_anatomy_default_budget(argcsr):  # test_argcsr.cpp:112-121
    m = argcsr.argcsr_from_csr(e8(argcsr), 12, 1)
    assert [(g.first_row, g.size, g.offset, g.chunk_size) for g in m.groups] == [(0, 7, 0, 1), (7, 1, 12, 2)]
    assert list(m.threads_mapping) == [1, 2, 3, 4, 5, 6, 7, 4]
    assert m.total_slots == 12 + 24


def test_chunk_entries_bounds(argcsr):  # test_argcsr.cpp:123-127
    m = argcsr.argcsr_from_csr(e8(argcsr), 12, 2)
    with pytest.raises(argcsr.BoundsError):
        argcsr.chunk_entries(m, 1, 0)
    with pytest.raises(argcsr.BoundsError):
        argcsr.chunk_entries(m, 0, 12)


def test_empty_rows_fully_padded(argcsr):  # test_argcsr.cpp:129-139
    a = argcsr.csr_from_triplets(4, 3, [(0, 0, 1.0), (0, 2, 2.0), (2, 1, 3.0)])
    m = argcsr.argcsr_from_csr(a, 4, 100)
    assert m.num_groups == 1 and m.groups[0].chunk_size == 2
    assert list(m.threads_mapping) == [1, 2, 3, 4]
    assert argcsr.chunk_entries(m, 0, 1) == [] and argcsr.chunk_entries(m, 0, 3) == []
    y = argcsr.spmv(m, [1.0, 1.0, 1.0])
    assert y == [3.0, 0.0, 3.0, 0.0]
    assert all(np.signbit(v) == False for v in y)  # +0.0 for empty rows  # noqa: E712


def test_all_zero_matrix(argcsr):  # test_argcsr.cpp:141-149
    a = argcsr.csr_from_triplets(3, 3, [])
    m = argcsr.argcsr_from_csr(a, 4, 1)
    assert m.num_groups == 1 and m.groups[0].chunk_size == 0 and m.total_slots == 0
    assert argcsr.spmv(m, [1.0, 1.0, 1.0]) == [0.0, 0.0, 0.0]
    assert argcsr.csr_from_argcsr(m) == a


def test_spmv_validates_length(argcsr):  # test_argcsr.cpp:217-220
    m = argcsr.argcsr_from_csr(e8(argcsr), 12, 2)
    with pytest.raises(argcsr.DimensionError):
        argcsr.spmv(m, [1.0] * 7)


def test_parameter_errors(argcsr):  # test_argcsr.cpp:32-36 via the converter
    with pytest.raises(argcsr.ParameterError):
        argcsr.argcsr_from_csr(e8(argcsr), 0, 1)
    with pytest.raises(argcsr.ParameterError):
        argcsr.argcsr_from_csr(e8(argcsr), 4, 0)


def test_padding_shrinks_with_threads(argcsr):  # test_argcsr.cpp:222-237
    a = e8(argcsr)
    padded = [argcsr.padding_stats(argcsr.argcsr_from_csr(a, t, 8)).assigned_padded_slots for t in range(8, 41)]
    assert padded[:5] == [49, 21, 15, 7, 7]
    assert all(padded[i] <= padded[i - 1] for i in range(1, len(padded)))


def test_padding_jump_14_15(argcsr):  # test_argcsr.cpp:239-249
    a = e8(argcsr)
    narrow = argcsr.padding_stats(argcsr.argcsr_from_csr(a, 14, 1))
    assert (narrow.assigned_padded_slots, narrow.total_allocated_slots) == (0, 42)
    wide = argcsr.padding_stats(argcsr.argcsr_from_csr(a, 15, 1))
    assert (wide.assigned_padded_slots, wide.total_allocated_slots) == (7, 30)


def test_e8_padding_smoke(argcsr):  # python/test_smoke.py:39-48
    s = argcsr.padding_stats(argcsr.argcsr_from_csr(e8(argcsr), threads_per_group=12, desired_chunk_size=2))
    assert (s.assigned_padded_slots, s.total_allocated_slots, s.explicit_nnz) == (7, 24, 15)


def test_spmv_agrees_with_reference_e8(argcsr, orc):  # python/test_smoke.py:21-30
    a = e8(argcsr)
    x = [1.0 + 0.25 * j for j in range(8)]
    A = Csr(8, 8, a.row_pointers, a.columns, a.values)
    y = argcsr.spmv(argcsr.argcsr_from_csr(a, threads_per_group=12, desired_chunk_size=2), x)
    assert y == list(orc.spmv_csr(A, x))
    assert y[7] == pytest.approx(sum(x))


# ------------------------------------------------------------ corpus x grid
GRID = [(t, d) for t in (1, 3, 4, 12, 32, 128) for d in (1, 2, 4, 32)]


def _check_case(argcsr, orc, A, tpg, dcs, where, layouts=LAYOUTS):
    """Both device layouts: exported arrays byte-equal to the oracle's, SpMV
    bit-identical to the reference order and within the north_star bound."""
    ref_m = orc.argcsr_from_csr(A, tpg, dcs)
    x = np.linspace(-1.5, 2.5, A.num_cols) if A.num_cols > 1 else np.array([1.25])
    y_ref = orc.spmv_argcsr(ref_m, x)
    y_csr = orc.spmv_csr(A, x)
    for layout in layouts:
        dev = to_dev(argcsr, A, tpg, dcs, layout=layout)
        w = f"{where} [{layout}]"
        assert dev.layout == layout[0]
        assert_same_layout(dev, ref_m, w)
        if layout[0] == "reference":
            assert dev.stored_slots == dev.total_slots and not dev.x_remap
        if layout == ("compact", "on") and A.columns.size:
            assert dev.x_remap and dev.x_used_columns == np.unique(A.columns).size
        else:
            assert dev.stored_slots <= dev.total_slots
        y = argcsr.spmv(dev, x)
        assert bits(y) == bits(y_ref), f"{w}: SpMV not bit-identical"
        assert within_bound(y, y_csr, orc.abs_row_sums(A, x), FP64_TOL), f"{w}: outside 1e-12 bound"
    return dev


def test_reference_corpus_grid(argcsr, orc, corpus):
    """All 500 reference corpus matrices x tpg {1,3,4,12,32,128} x dcs {1,2,4,32}."""
    for i, A in enumerate(corpus):
        for tpg, dcs in GRID:
            _check_case(argcsr, orc, A, tpg, dcs, f"corpus[{i}] ({tpg},{dcs})")


def test_numpy_corpus_grid(argcsr, orc):
    for i, A in enumerate(np_corpus(120)):
        for tpg, dcs in ((4, 1), (32, 4), (128, 1), (128, 32), (100, 3), (30, 2), (127, 1)):
            _check_case(argcsr, orc, A, tpg, dcs, f"np_corpus[{i}] ({tpg},{dcs})")


def test_round_trip_corpus(argcsr, corpus):  # test_argcsr.cpp:190-201, acceptance criterion 4
    for A in corpus[:100]:
        for (tpg, dcs), layout in zip(((4, 1), (32, 4), (128, 32), (128, 1)), LAYOUTS * 2):
            m = to_dev(argcsr, A, tpg, dcs, layout=layout)
            rp, cols, vals = argcsr.csr_arrays_from_argcsr(m)
            assert np.array_equal(rp, A.row_pointers)
            assert np.array_equal(cols, A.columns)
            assert vals.tobytes() == A.values.tobytes()


def test_skew_and_uniform_families(argcsr, orc, ref):  # acceptance.cpp:171-198
    for k in range(1, 33):
        A = ref.skew(k)
        for tpg, dcs in ((128, 1), (128, 32), (12, 2)):
            _check_case(argcsr, orc, A, tpg, dcs, f"skew({k}) ({tpg},{dcs})")
        assert to_dev(argcsr, A, 128, 1).total_slots <= to_dev(argcsr, A, 128, 32).total_slots
    U = ref.uniform(128, 128, 4)
    assert to_dev(argcsr, U, 32, 32).num_groups <= to_dev(argcsr, U, 32, 1).num_groups
    _check_case(argcsr, orc, U, 32, 1, "uniform")


# --------------------------------------------------------- larger / edge cases
@pytest.mark.parametrize("heavy", ["default", "ARGCSR_HEAVY_PIPE=1", "ARGCSR_LIGHT_DYN=0", "ARGCSR_LIGHT_DYN=1"])
@pytest.mark.parametrize("tpg,dcs", [(128, 1), (128, 4), (64, 2), (32, 1), (100, 1), (30, 3), (127, 1), (256, 1)])
def test_powerlaw_heavy_groups(argcsr, orc, tpg, dcs, heavy, monkeypatch):
    """Heavy-tailed rows: long-chunk (heavy) groups, multi-tile schedule,
    through two heavy-kernel variants."""
    if heavy != "default":
        for kv in heavy.split(","):
            monkeypatch.setenv(*kv.split("="))
        argcsr._ext.reload_options()
    A = powerlaw_csr(40000, 30000, seed=tpg * 7 + dcs, heavy_rows=[(0, 25000), (777, 12000), (39999, 9000)])
    dev = _check_case(argcsr, orc, A, tpg, dcs, f"powerlaw ({tpg},{dcs})")
    assert dev.heavy_groups > 0


@pytest.mark.parametrize("layout_opt", ["auto", "ARGCSR_VEC=4"])
def test_powerlaw_schedule_one_lane_units(argcsr, orc, layout_opt, monkeypatch):
    """Power-law matrices (heavy groups AND light lanes of >= 8 steps) run the
    light tiles one lane per unit over 2048-unit tiles (convert.cu
    powerlaw_schedule): the stored lane stride is then the assigned lane count
    itself, not rounded up to 4.  Bit-exact either way."""
    if layout_opt != "auto":
        monkeypatch.setenv(*layout_opt.split("="))
        argcsr._ext.reload_options()
    A = powerlaw_csr(60000, 60000, seed=31, heavy_rows=[(5, 30000), (40000, 20000)])
    M = orc.argcsr_from_csr(A, 128, 1)
    G = np.asarray(M.groups).reshape(-1, 4).astype(np.int64)
    tm = np.asarray(M.threads_mapping).astype(np.int64)
    last = np.concatenate([G[1:, 0], [A.num_rows]]) - 1
    assigned, chunk = tm[last], G[:, 3]
    assert chunk.max() > 32 and chunk[chunk <= 32].max() >= 8  # the schedule's precondition
    _check_case(argcsr, orc, A, 128, 1, f"powerlaw schedule ({layout_opt})")
    dev = to_dev(argcsr, A, 128, 1)  # lane-compact, x remap auto
    exact = int((chunk * assigned).sum())
    rounded = int((chunk * ((assigned + 3) // 4 * 4)).sum())
    assert exact < rounded
    assert dev.stored_slots == (exact if layout_opt == "auto" else rounded)


@pytest.mark.parametrize("tpg", [1, 2, 1024, 1025, 4000, 16384])
def test_extreme_threads_per_group(argcsr, orc, tpg):
    """tpg > 1024 takes the sequential group walk; 16384 is the device limit."""
    A = powerlaw_csr(3000, 2000, seed=tpg, max_len=1500)
    _check_case(argcsr, orc, A, tpg, 1, f"tpg={tpg}")


def test_threads_per_group_limit(argcsr):
    with pytest.raises(argcsr.UnsupportedError):
        argcsr.argcsr_from_csr(e8(argcsr), 16385, 1)


def test_budget_wraps_like_size_t(argcsr, orc):
    """desired_chunk_size * threads_per_group overflows size_t exactly as in argcsr.cpp:28."""
    A = powerlaw_csr(500, 400, seed=3, max_len=300)
    for dcs in (2**62, 2**63 + 5, 2**64 - 1):
        _check_case(argcsr, orc, A, 4, dcs, f"dcs={dcs}")


@pytest.mark.parametrize("n,params", [(24, [(128, 1), (128, 32), (128, 4)]), (61, [(128, 1), (128, 32)])])
def test_stencil27(argcsr, orc, n, params):
    A = stencil27(n)
    for tpg, dcs in params:
        _check_case(argcsr, orc, A, tpg, dcs, f"stencil27({n}) ({tpg},{dcs})")


def test_rectangular_and_single_column(argcsr, orc):
    rng = np.random.default_rng(5)
    for nr, nc in ((1, 1), (1, 500), (700, 1), (5, 9000), (20000, 3)):
        dens = min(1.0, 8.0 / nc)
        mask = rng.random((nr, nc)) < dens
        r, c = np.nonzero(mask)
        rp = np.zeros(nr + 1, np.uint64)
        np.add.at(rp, r + 1, 1)
        A = Csr(nr, nc, np.cumsum(rp).astype(np.uint64), c.astype(np.int32), rng.uniform(-1, 1, c.size))
        for tpg, dcs in ((128, 1), (4, 1), (32, 32)):
            _check_case(argcsr, orc, A, tpg, dcs, f"{nr}x{nc} ({tpg},{dcs})")


def test_unsorted_columns_copied_in_stored_order(argcsr, orc):
    """The converter neither validates nor re-sorts (argcsr.cpp:107-117)."""
    rp = np.array([0, 3, 3, 7], np.uint64)
    cols = np.array([2, 0, 1, 4, 4, 0, 3], np.int32)
    vals = np.array([1.5, -2.0, 0.25, 3.0, 1.0, -0.5, 2.0])
    A = Csr(3, 5, rp, cols, vals)
    for tpg, dcs in ((4, 1), (2, 1), (12, 2)):
        _check_case(argcsr, orc, A, tpg, dcs, f"unsorted ({tpg},{dcs})")


# ---------------------------------------------------------------- other APIs
@pytest.mark.parametrize("layout", LAYOUTS)
@pytest.mark.parametrize("heavy", ["default", "ARGCSR_HEAVY_PIPE=1", "ARGCSR_HEAVY_PIPE=0"])
def test_spmv_groups_writes_only_its_rows(argcsr, orc, layout, heavy, monkeypatch):
    import torch

    if heavy != "default":
        for kv in heavy.split(","):
            monkeypatch.setenv(*kv.split("="))
        argcsr._ext.reload_options()

    A = powerlaw_csr(20000, 20000, seed=11, heavy_rows=[(100, 8000)])
    ref_m = orc.argcsr_from_csr(A, 128, 1)
    dev = to_dev(argcsr, A, 128, 1, layout=layout)
    x = np.cos(np.arange(A.num_cols, dtype=np.float64))
    G = dev.num_groups
    for gb, ge in ((0, G), (3, G // 2), (G // 3, G - 1), (5, 6)):
        y = torch.full((A.num_rows,), 7.0, dtype=torch.float64, device="cuda")
        argcsr.spmv_argcsr_groups(dev, torch.from_numpy(x).cuda(), gb, ge, y)
        y_ref = np.full(A.num_rows, 7.0)
        orc.lib.orc_spmv_argcsr_groups  # same semantics as argcsr.cpp:185-217
        full = orc.spmv_argcsr(ref_m, x)
        r0 = int(ref_m.groups[gb, 0]) if gb < G else A.num_rows
        r1 = int(ref_m.groups[ge, 0]) if ge < G else A.num_rows
        y_ref[r0:r1] = full[r0:r1]
        assert bits(y.cpu().numpy()) == bits(y_ref), f"groups [{gb},{ge})"


@pytest.mark.parametrize("policy", ["ARGCSR_L2PF=0", "ARGCSR_L2PF=1,ARGCSR_L2PF_WHAT=b",
                                    "ARGCSR_L2PF=1,ARGCSR_L2PF_WHAT=c,ARGCSR_XPOL=0",
                                    "ARGCSR_L2PF=2,ARGCSR_L2PF_WHAT=v,ARGCSR_XPOL=1"])
def test_l2_policy_variants(argcsr, orc, policy, monkeypatch):
    """The light tiles' L2 prefetch (spmv.cu tile_prefetch_l2: forced off; on
    for both arrays; columns only with evict_normal x; values only with a 2 KB
    tile bound) only moves lines into L2: results stay bit-identical,
    including group sub-ranges (the prefetch then follows the range check)."""
    import torch

    for kv in policy.split(","):
        monkeypatch.setenv(*kv.split("="))
    argcsr._ext.reload_options()
    A = stencil27(40)
    for tpg, dcs in ((128, 1), (128, 4), (32, 1)):
        _check_case(argcsr, orc, A, tpg, dcs, f"stencil27(40) ({tpg},{dcs}) {policy}")
    P = powerlaw_csr(30000, 30000, seed=4, heavy_rows=[(17, 12000)])
    _check_case(argcsr, orc, P, 128, 1, f"powerlaw {policy}")
    ref_m = orc.argcsr_from_csr(A, 128, 1)
    dev = to_dev(argcsr, A, 128, 1)
    x = np.cos(np.arange(A.num_cols, dtype=np.float64))
    full = orc.spmv_argcsr(ref_m, x)
    G = dev.num_groups
    for gb, ge in ((0, G), (7, G // 2), (G // 3, G)):
        y = torch.full((A.num_rows,), 7.0, dtype=torch.float64, device="cuda")
        argcsr.spmv_argcsr_groups(dev, torch.from_numpy(x).cuda(), gb, ge, y)
        y_ref = np.full(A.num_rows, 7.0)
        r0 = int(ref_m.groups[gb, 0])
        r1 = int(ref_m.groups[ge, 0]) if ge < G else A.num_rows
        y_ref[r0:r1] = full[r0:r1]
        assert bits(y.cpu().numpy()) == bits(y_ref), f"groups [{gb},{ge}) {policy}"


def test_padding_stats_matches_reference(argcsr, orc, ref, corpus):
    for A in corpus[:60]:
        for (tpg, dcs), layout in ((t, l) for t in ((4, 1), (32, 4), (128, 1)) for l in LAYOUTS):
            m = to_dev(argcsr, A, tpg, dcs, layout=layout)
            want = ref.padding_stats(orc.argcsr_from_csr(A, tpg, dcs))
            got = argcsr.padding_stats(m)
            assert got.explicit_nnz == want["explicit_nnz"]
            assert got.assigned_padded_slots == want["assigned_padded_slots"]
            assert got.total_allocated_slots == want["total_allocated_slots"]
            assert got.estimated_bytes == want["estimated_bytes"]
            assert (got.padding_ratio == want["padding_ratio"]) or (
                np.isinf(got.padding_ratio) and np.isinf(want["padding_ratio"]))


def test_chunk_entries_match_reference(argcsr, orc, ref, corpus):
    for A in corpus[1:30]:
        ref_m = orc.argcsr_from_csr(A, 32, 4)
        for layout in LAYOUTS:
            m = to_dev(argcsr, A, 32, 4, layout=layout)
            for g in range(0, m.num_groups, max(1, m.num_groups // 5)):
                for c in (0, 5, 31):
                    assert argcsr.chunk_entries(m, g, c) == ref.chunk_entries(ref_m, g, c), (layout, g, c)


def test_determinism(argcsr):
    import torch

    A = powerlaw_csr(50000, 50000, seed=2, heavy_rows=[(9, 30000)])
    m = to_dev(argcsr, A, 128, 1)
    x = torch.rand(A.num_cols, dtype=torch.float64, device="cuda")
    y1 = argcsr.spmv_torch(m, x).cpu().numpy()
    for _ in range(3):
        assert bits(argcsr.spmv_torch(m, x).cpu().numpy()) == bits(y1)


def test_fp32_handle(argcsr, orc):
    """fp32 values/x: exact fp64 products, one rounding per row -> equals the
    fp64 reference on fp32-representable inputs, rounded (bound 1e-5)."""
    A = powerlaw_csr(30000, 25000, seed=9, heavy_rows=[(4, 20000)])
    A32 = Csr(A.num_rows, A.num_cols, A.row_pointers, A.columns, A.values.astype(np.float32).astype(np.float64))
    x32 = np.sin(np.arange(A.num_cols)).astype(np.float32)
    for (tpg, dcs), layout in ((t, l) for t in ((128, 1), (128, 8), (32, 1)) for l in LAYOUTS):
        ref_m = orc.argcsr_from_csr(A32, tpg, dcs)
        dev = to_dev(argcsr, A32, tpg, dcs, dtype=np.float32, layout=layout)
        assert dev.dtype == "float32"
        assert np.array_equal(dev.groups_array, ref_m.groups)
        assert np.array_equal(dev.threads_mapping, ref_m.threads_mapping)
        assert np.array_equal(dev.columns, ref_m.columns)
        assert np.array_equal(dev.values, ref_m.values.astype(np.float32))
        y = argcsr.spmv(dev, x32)
        assert y.dtype == np.float32
        y64 = orc.spmv_argcsr(ref_m, x32.astype(np.float64))
        assert np.array_equal(y, y64.astype(np.float32))
        absrow = orc.abs_row_sums(A32, x32.astype(np.float64))
        assert within_bound(y, orc.spmv_csr(A32, x32.astype(np.float64)), absrow, FP32_TOL)


def test_torch_device_path(argcsr, orc):
    import torch

    A = stencil27(20)
    dev = argcsr.argcsr_from_torch(
        A.num_rows, A.num_cols, torch.from_numpy(A.row_pointers.astype(np.int64)).cuda(),
        torch.from_numpy(A.columns).cuda(), torch.from_numpy(A.values).cuda(), 128, 1)
    assert_same_layout(dev, orc.argcsr_from_csr(A, 128, 1), "torch input")
    x = torch.linspace(0, 1, A.num_cols, dtype=torch.float64, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        y = argcsr.spmv_torch(dev, x)
    s.synchronize()
    assert bits(y.cpu().numpy()) == bits(orc.spmv_argcsr(orc.argcsr_from_csr(A, 128, 1), x.cpu().numpy()))
    with pytest.raises(argcsr.DimensionError):
        argcsr.spmv_torch(dev, x[:-1])


HEAVY_VARIANTS = ["default", "ARGCSR_HEAVY_PIPE=1", "ARGCSR_HEAVY_PIPE=0"]


@pytest.mark.parametrize("heavy", HEAVY_VARIANTS)
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("layout", LAYOUTS)
def test_dense_rows_vector_x_runs(argcsr, orc, dtype, layout, heavy, monkeypatch):
    """Long rows whose columns run consecutively (directly, or after the x
    remap for strided dense rows), through every heavy-kernel variant (the
    default scalar gathers, vector x loads over runs, 4/16 steps in flight);
    results stay bit-identical (fp32: one rounding of the fp64 sum)."""
    if heavy != "default":
        for kv in heavy.split(","):
            monkeypatch.setenv(*kv.split("="))
        argcsr._ext.reload_options()
    rng = np.random.default_rng(3)
    n = 6000
    rows, cols = [], []
    for r in range(n):
        if r % 1500 == 7:
            c = np.arange(0, n, 3) if r % 3000 == 7 else np.arange(r % 11, n - 5)  # strided / consecutive dense rows
        else:
            c = np.unique(np.clip(r + rng.integers(-3, 4, 3), 0, n - 1))
        rows.append(np.full(c.size, r))
        cols.append(c)
    r_ = np.concatenate(rows)
    c_ = np.concatenate(cols).astype(np.int32)
    rp = np.zeros(n + 1, np.uint64)
    np.add.at(rp, r_ + 1, 1)
    vals = rng.uniform(-1, 1, c_.size)
    if dtype == np.float32:
        vals = vals.astype(np.float32).astype(np.float64)
    A = Csr(n, n, np.cumsum(rp).astype(np.uint64), c_, vals)
    ref_m = orc.argcsr_from_csr(A, 128, 1)
    dev = to_dev(argcsr, A, 128, 1, dtype=dtype, layout=layout)
    assert dev.heavy_groups > 0
    x = np.sin(np.arange(n)).astype(dtype)
    y = argcsr.spmv(dev, x)
    y_ref = orc.spmv_argcsr(ref_m, x.astype(np.float64))
    if dtype == np.float64:
        assert bits(y) == bits(y_ref)
    else:
        assert np.array_equal(y, y_ref.astype(np.float32))


@pytest.mark.parametrize("kind", ["stencil", "powerlaw"])
def test_host_staged_pipeline(argcsr, orc, kind):
    """argcsr_dev_spmv_host_staged (the e2e path): x up in pieces, tiles as
    soon as their columns have arrived, y down in chunks (banded matrices);
    one-shot otherwise.  Bit-identical to the reference either way."""
    import torch

    A = stencil27(30) if kind == "stencil" else powerlaw_csr(30000, 30000, seed=12, heavy_rows=[(5, 9000)])
    dev = to_dev(argcsr, A, 128, 1)
    x = np.sin(np.arange(A.num_cols, dtype=np.float64))
    xh = torch.from_numpy(x).pin_memory()
    yh = torch.empty(A.num_rows, dtype=torch.float64).pin_memory()
    xd = torch.empty(A.num_cols, dtype=torch.float64, device="cuda")
    yd = torch.empty(A.num_rows, dtype=torch.float64, device="cuda")
    s = torch.cuda.Stream()
    for _ in range(2):
        dev.spmv_host_staged(xh.data_ptr(), xd.data_ptr(), yd.data_ptr(), yh.data_ptr(), s.cuda_stream)
        assert bits(yh.numpy()) == bits(orc.spmv_argcsr(orc.argcsr_from_csr(A, 128, 1), x))


@pytest.mark.parametrize("ulen", ["1", "0"])
def test_unit_lengths_forced(argcsr, orc, corpus, monkeypatch, ulen):
    """Light units stop at their stored length (the u8 unit-length table) or
    read to the group's chunk: both bit-identical to the reference order."""
    monkeypatch.setenv("ARGCSR_ULEN", ulen)
    argcsr._ext.reload_options()
    cases = [(A, t, d, f"corpus[{i}]") for i, A in enumerate(corpus[:60]) for t, d in ((4, 1), (12, 2), (128, 1), (32, 4))]
    cases += [(powerlaw_csr(40000, 30000, seed=11, heavy_rows=[(5, 20000)]), t, d, "powerlaw")
              for t, d in ((128, 1), (128, 4), (64, 2))]
    cases += [(stencil27(12), 128, 1, "stencil27(12)")]
    for A, tpg, dcs, w in cases:
        dev = _check_case(argcsr, orc, A, tpg, dcs, f"{w} ({tpg},{dcs}) ulen={ulen}", layouts=(("compact", "auto"), ("reference", "auto")))
        if ulen == "0":
            assert dev.unit_len_bytes == 0
        elif A.nnz:
            assert dev.unit_len_bytes > 0


@pytest.mark.parametrize("kind", ["stencil", "powerlaw", "remap"])
def test_host_async_stream(argcsr, orc, kind):
    """argcsr_dev_spmv_host_async: a stream of calls with different x and y
    host buffers, overlapped through the handle's double-buffered staging;
    after argcsr_dev_host_wait every y is the oracle's, bit for bit."""
    import torch

    if kind == "stencil":
        A = stencil27(12)
    else:
        A = powerlaw_csr(20000, 20000, seed=21, heavy_rows=[(4, 9000)])
    dev = to_dev(argcsr, A, 128, 1, layout=("compact", "on") if kind == "remap" else "compact")
    ref_m = orc.argcsr_from_csr(A, 128, 1)
    xs = [torch.from_numpy(np.cos(np.arange(A.num_cols) * (0.1 + i))).pin_memory() for i in range(5)]
    ys = [torch.empty(A.num_rows, dtype=torch.float64).pin_memory() for _ in range(5)]
    s = torch.cuda.current_stream().cuda_stream
    for x, y in zip(xs, ys):
        dev.spmv_host_async(x.data_ptr(), y.data_ptr(), s)
    dev.host_wait()
    for x, y in zip(xs, ys):
        assert bits(y.numpy()) == bits(orc.spmv_argcsr(ref_m, x.numpy()))


def test_balance_stats_matches_reference(argcsr, ref, corpus):
    """balance_stats (analysis.cpp:198-208): per-group explicit entries equal,
    max/mean and the coefficient of variation bit-identical to the compiled
    reference, in both device layouts and with heavy groups."""
    cases = [(A, t, d) for A in corpus[:80] for t, d in ((4, 1), (32, 4), (128, 1))]
    cases += [(powerlaw_csr(20000, 20000, seed=3, heavy_rows=[(1, 9000)]), 128, 1), (stencil27(10), 128, 32)]
    for A, tpg, dcs in cases:
        per_ref, mom_ref, cv_ref = ref.balance_stats(ref.argcsr_from_csr(A, tpg, dcs))
        for layout in ("compact", "reference"):
            b = argcsr.balance_stats(to_dev(argcsr, A, tpg, dcs, layout=layout))
            assert np.array_equal(np.asarray(b.per_group_nnz, np.uint64), per_ref)
            assert bits(np.array([b.max_over_mean, b.coefficient_of_variation])) == bits(np.array([mom_ref, cv_ref]))
