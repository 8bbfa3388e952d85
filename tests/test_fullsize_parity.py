"""Full-size conversion parity: the device converter against the compiled
reference (oracle/_ref = the unmodified proj/src/argcsr.cpp:123-155
argcsr_from_csr) on the BASELINE.json configurations themselves.

For every case the SAME CSR (workloads.py, generated on the device, copied to
the host) goes through both converters and all four reference arrays are
compared byte for byte (groups, threads_mapping, values, columns), then the
device SpMV is compared bit for bit with the reference spmv_argcsr_parallel
on the reference's own conversion.  The cases also drive the converter's
multi-batch paths that small matrices never reach: k2_resolve composes the
per-tile transfer tables in shared-memory batches of kResolveBatch / tpg
tiles (93 tiles = ~762k rows at tpg 128, 11 tiles = ~90k rows at tpg 1024,
csrc/convert.cu), so every case here runs through 3+ batches.
"""
from __future__ import annotations

import numpy as np
import pytest

import oracle

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def _host_csr(A) -> oracle.Csr:
    return oracle.Csr(A.num_rows, A.num_cols, A.row_pointers.cpu().numpy().view(np.uint64),
                      A.columns.cpu().numpy(), A.values.cpu().numpy())


def _check(argcsr, ref, A, tpg: int, dcs: int, spmv: bool = True) -> dict:
    import torch

    import workloads

    m = argcsr.argcsr_from_torch(A.num_rows, A.num_cols, A.row_pointers, A.columns, A.values, tpg, dcs)
    H = _host_csr(A)
    h = ref.argcsr_handle(H, tpg, dcs)
    try:
        R = ref.export(h)
        where = f"{A.name} (tpg={tpg}, dcs={dcs})"
        assert m.num_groups == R.groups.shape[0], f"{where}: groups {m.num_groups} != {R.groups.shape[0]}"
        assert m.total_slots == R.total_slots, f"{where}: total slots {m.total_slots} != {R.total_slots}"
        assert np.array_equal(m.groups_array, R.groups), f"{where}: groups differ"
        assert np.array_equal(np.asarray(m.threads_mapping), R.threads_mapping), f"{where}: threads_mapping differs"
        cols = np.asarray(m.columns)
        assert np.array_equal(cols, R.columns), f"{where}: columns differ"
        del cols
        vals = np.asarray(m.values)
        assert np.array_equal(vals.view(np.uint64), R.values.view(np.uint64)), f"{where}: values differ"
        del vals
        out = {"groups": m.num_groups, "slots": m.total_slots}
        del R
        if spmv:
            x = workloads.bench_input(A.num_cols, "cuda")
            y = argcsr.spmv(m, x)
            torch.cuda.synchronize()
            _, y_ref = ref.time_spmv_argcsr_parallel(h, x.cpu().numpy(), ref.hardware_threads(), 0, 1, A.num_rows)
            assert y.cpu().numpy().tobytes() == y_ref.tobytes(), f"{where}: SpMV not bit-identical"
        return out
    finally:
        ref.free_argcsr(h)
        m.free()


@pytest.mark.parametrize("dcs", [1, 32])
def test_c1_stencil2d5_1024(argcsr, ref, dcs):
    import workloads

    A = workloads.stencil2d5(1024, "cuda")
    out = _check(argcsr, ref, A, 128, dcs)
    if dcs == 1:  # SURVEY §8(a) a4/a8 probe numbers
        assert (out["groups"], out["slots"]) == (41885, 10722560)


@pytest.mark.parametrize("dcs", [1, 32])
def test_c2_stencil3d27_160(argcsr, ref, dcs):
    import workloads

    A = workloads.stencil3d27(160, "cuda")
    out = _check(argcsr, ref, A, 128, dcs)
    if dcs == 1:
        assert (out["groups"], out["slots"]) == (1004741, 512584576)
    else:
        assert out["slots"] == 109764096


def test_c4_arrowhead(argcsr, ref):
    import workloads

    A = workloads.arrowhead(device="cuda")
    out = _check(argcsr, ref, A, 128, 1)
    assert (out["groups"], out["slots"]) == (225295, 262147840)


def test_rmat_scale22_heavy_rows(argcsr, ref):
    """R-MAT 2^22 (4.2M rows, ~67M nnz): power-law rows up to tens of
    thousands of entries (heavy groups), many empty rows."""
    import workloads

    A = workloads.rmat(22, 16, 1, "cuda")
    _check(argcsr, ref, A, 128, 1)


def _ragged(rows: int, seed: int, max_len: int = 9):
    """A >2M-row matrix with row lengths 0..max_len-1 (empty rows included),
    random columns (unsorted within rows: the converter must not sort)."""
    import torch

    import workloads

    g = torch.arange(rows, device="cuda", dtype=torch.int64)
    lens = (workloads._srl(workloads.hash_stream(seed, g), 40) % max_len)
    rp = torch.zeros(rows + 1, dtype=torch.int64, device="cuda")
    torch.cumsum(lens, 0, out=rp[1:])
    nnz = int(rp[-1])
    k = torch.arange(nnz, device="cuda", dtype=torch.int64)
    cols = (workloads._srl(workloads.hash_stream(seed + 1, k), 20) % rows).to(torch.int32)
    vals = workloads.uniform_pm1(seed + 2, k)
    return workloads.SynthCsr(f"ragged_{rows}", rows, rows, rp, cols, vals)


def test_multibatch_resolve_tpg128(argcsr, ref):
    A = _ragged(3_000_000, 11)  # ~366 tiles of 8192 rows: 4 resolve batches at tpg 128
    _check(argcsr, ref, A, 128, 1)
    _check(argcsr, ref, A, 128, 4, spmv=False)


def test_multibatch_resolve_tpg1024(argcsr, ref):
    A = _ragged(400_000, 12, max_len=40)  # 49 tiles: 5 resolve batches at tpg 1024
    _check(argcsr, ref, A, 1024, 1)
    _check(argcsr, ref, A, 1024, 3, spmv=False)


def test_tpg4_tpg1024_stencil(argcsr, ref):
    import workloads

    A = workloads.stencil3d27(100, "cuda")  # 1M rows, 26.5M nnz
    _check(argcsr, ref, A, 4, 1)
    _check(argcsr, ref, A, 1024, 1)
    _check(argcsr, ref, A, 1024, 8, spmv=False)
