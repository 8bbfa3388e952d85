"""ELLPACK and Sliced ELLPACK on the device (the paper's comparison formats,
proj/src/ellpack.cpp) against the compiled reference: the stored arrays are
byte-equal to ellpack_from_csr / sliced_from_csr, the SpMV is bit-identical to
spmv_ellpack / spmv_sliced (same order: j ascending from +0.0, stop at the
first padding slot), and csr_from_* round-trips (ellpack.cpp:62-119)."""
import numpy as np
import pytest

from helpers import bits, powerlaw_csr, stencil27

pytestmark = pytest.mark.gpu


def _csr(argcsr, A):
    return argcsr.CsrMatrix.from_arrays(A.num_rows, A.num_cols, A.row_pointers, A.columns, A.values)


def _cases(corpus):
    return list(corpus[:120]) + [stencil27(12), powerlaw_csr(3000, 2500, seed=8, max_len=400)]


def test_ellpack_matches_reference(argcsr, ref, corpus):
    for i, A in enumerate(_cases(corpus)):
        x = np.linspace(-1, 1, A.num_cols) if A.num_cols > 1 else np.array([0.5])
        width, vals, cols, y_ref = ref.ellpack(A, x)
        M = argcsr.ellpack_from_csr(_csr(argcsr, A))
        assert M.width == width and M.total_slots == vals.size, i
        assert np.array_equal(M.columns, cols) and M.values.tobytes() == vals.tobytes(), i
        assert bits(argcsr.spmv(M, x)) == bits(y_ref), i
        B = argcsr.csr_from_ellpack(M)
        assert np.array_equal(B.row_pointers, A.row_pointers) and np.array_equal(B.columns, A.columns), i


@pytest.mark.parametrize("slice_size", [1, 3, 32, 100])
def test_sliced_matches_reference(argcsr, ref, corpus, slice_size):
    for i, A in enumerate(_cases(corpus)):
        x = np.cos(np.arange(A.num_cols, dtype=np.float64))
        w, o, vals, cols, y_ref = ref.sliced(A, slice_size, x)
        M = argcsr.sliced_from_csr(_csr(argcsr, A), slice_size)
        assert M.num_slices() == w.size and np.array_equal(M.slice_widths, w), i
        assert np.array_equal(M.slice_offsets, o), i
        assert np.array_equal(M.columns, cols) and M.values.tobytes() == vals.tobytes(), i
        assert bits(argcsr.spmv(M, x)) == bits(y_ref), i
        B = argcsr.csr_from_sliced(M)
        assert np.array_equal(B.row_pointers, A.row_pointers) and B.values.tobytes() == A.values.tobytes(), i


def test_errors_and_torch_path(argcsr, ref, corpus):
    import torch

    A = corpus[5]
    with pytest.raises(argcsr.ParameterError):
        argcsr.sliced_from_csr(_csr(argcsr, A), 0)
    M = argcsr.sliced_from_csr(_csr(argcsr, A), 32)
    with pytest.raises(argcsr.DimensionError):
        argcsr.spmv(M, np.zeros(A.num_cols + 1))
    x = torch.linspace(0, 1, A.num_cols, dtype=torch.float64, device="cuda")
    y = argcsr.spmv_torch(M, x)
    assert bits(y.cpu().numpy()) == bits(ref.sliced(A, 32, x.cpu().numpy())[4])
