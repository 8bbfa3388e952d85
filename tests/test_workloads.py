"""The bench / test inputs (workloads.py) are pure functions of their
arguments and identical on every device, so both bench arms and every test
time and check the same matrices.  Digests pinned here were produced on the
CPU; the GPU test regenerates them on cuda:0."""
import numpy as np
import pytest

import workloads

PINNED = {
    "rmat14": ("21a3320e3eba8e6b", lambda d: workloads.rmat(14, 16, 1, d)),
    "arrow": ("5960a490fd901402", lambda d: workloads.arrowhead(20000, 16, 2000, 7, d)),
    "st27": ("df9c6d5c2a18b536", lambda d: workloads.stencil3d27(12, d)),
    "st5": ("98c0cfc8f21ac4cd", lambda d: workloads.stencil2d5(30, d)),
}


@pytest.mark.parametrize("name", sorted(PINNED))
def test_pinned_digest_cpu(name):
    digest, gen = PINNED[name]
    assert gen("cpu").digest() == digest


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(PINNED))
def test_same_matrix_on_gpu(name):
    digest, gen = PINNED[name]
    assert gen("cuda").digest() == digest


def test_csr_invariants_cpu():
    """core.hpp:24-30: rp[0] = 0, non-decreasing, strictly increasing columns
    per row (the generators' rows are sorted and duplicate-free)."""
    for _, gen in PINNED.values():
        A = gen("cpu")
        rp = A.row_pointers.numpy()
        c = A.columns.numpy().astype(np.int64)
        assert rp[0] == 0 and np.all(np.diff(rp) >= 0) and rp[-1] == c.size
        row = np.repeat(np.arange(A.num_rows), np.diff(rp))
        same = row[1:] == row[:-1]
        assert np.all(c[1:][same] > c[:-1][same])
        assert c.min() >= 0 and c.max() < A.num_cols
        v = A.values.numpy()
        assert np.all(np.abs(v) <= 26.0)


def test_hash_matches_splitmix64():
    import torch

    M = (1 << 64) - 1

    def mix(z):
        z &= M
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
        return z ^ (z >> 31)

    idx = [0, 1, 2, 12345678901, 2**40 + 7]
    h = workloads.hash_stream(5, torch.tensor(idx, dtype=torch.int64)).tolist()
    for i, v in zip(idx, h):
        assert v & M == mix(i * 0x9E3779B97F4A7C15 + ((5 * 0xD1B54A32D192ED03 + 1) & M))


def test_uniform_range():
    import torch

    v = workloads.uniform_pm1(3, torch.arange(100000, dtype=torch.int64))
    assert float(v.min()) >= -1.0 and float(v.max()) < 1.0 and abs(float(v.mean())) < 0.02
