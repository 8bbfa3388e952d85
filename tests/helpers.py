"""Shared test helpers: random corpora and device/oracle comparison."""
from __future__ import annotations

import numpy as np

import oracle
from oracle import Csr


def np_corpus(count: int, seed: int = 1203) -> list[Csr]:
    """A corpus shaped like proj/tests/support.hpp:86-119 (sizes 1..200,
    densities 0.5%..50%, forced empty rows, full rows, single-column matrices,
    one all-zero 3x3), drawn with numpy so it exists without oracle/_ref."""
    rng = np.random.default_rng(seed)
    out = [Csr(3, 3, np.zeros(4, np.uint64), np.zeros(0, np.int32), np.zeros(0))]
    while len(out) < count:
        idx = len(out)
        rows = int(rng.integers(1, 201))
        cols = 1 if idx % 13 == 0 else int(rng.integers(1, 201))
        density = rng.uniform(0.005, 0.5)
        mask = rng.random((rows, cols)) < density
        if idx % 7 == 0:
            mask[::5, :] = False
        if idx % 11 == 0:
            mask[rows // 2, :] = True
        r, c = np.nonzero(mask)
        rp = np.zeros(rows + 1, np.uint64)
        np.add.at(rp, r + 1, 1)
        rp = np.cumsum(rp).astype(np.uint64)
        out.append(Csr(rows, cols, rp, c.astype(np.int32), rng.uniform(-1, 1, c.size)))
    return out


def powerlaw_csr(rows: int, cols: int, seed: int, max_len: int = 5000, heavy_rows=()) -> Csr:
    """Heavy-tailed row lengths (exercises adaptive threads-per-row and the
    long-chunk path)."""
    rng = np.random.default_rng(seed)
    lens = np.minimum((rng.pareto(1.2, rows) * 3).astype(np.int64), max_len)
    lens = np.minimum(lens, cols)
    for r, n in heavy_rows:
        lens[r] = min(n, cols)
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint64)
    parts = [np.sort(rng.choice(cols, int(n), replace=False)) if n else np.zeros(0, np.int64) for n in lens]
    c = np.concatenate(parts).astype(np.int32) if parts else np.zeros(0, np.int32)
    return Csr(rows, cols, rp, c, rng.uniform(-1, 1, c.size))


def stencil27(n: int) -> Csr:
    """27-point stencil on an n^3 grid, ascending columns."""
    i, j, k = np.meshgrid(np.arange(n), np.arange(n), np.arange(n), indexing="ij")
    i, j, k = i.ravel(), j.ravel(), k.ravel()
    rows, colsl, valsl = [], [], []
    for di in (-1, 0, 1):
        for dj in (-1, 0, 1):
            for dk in (-1, 0, 1):
                ii, jj, kk = i + di, j + dj, k + dk
                ok = (ii >= 0) & (ii < n) & (jj >= 0) & (jj < n) & (kk >= 0) & (kk < n)
                r = ((i * n + j) * n + k)[ok]
                c = ((ii * n + jj) * n + kk)[ok]
                rows.append(r)
                colsl.append(c)
                valsl.append(np.full(r.size, 26.0 if di == dj == dk == 0 else -1.0))
    r = np.concatenate(rows)
    c = np.concatenate(colsl)
    v = np.concatenate(valsl)
    order = np.lexsort((c, r))
    r, c, v = r[order], c[order], v[order]
    rp = np.zeros(n**3 + 1, np.uint64)
    np.add.at(rp, r + 1, 1)
    return Csr(n**3, n**3, np.cumsum(rp).astype(np.uint64), c.astype(np.int32), v)


# device storage variants every parity case runs through: (layout, x_remap)
LAYOUTS = (("compact", "auto"), ("reference", "auto"), ("compact", "on"))


def to_dev(argcsr, A: Csr, tpg: int, dcs: int, dtype=np.float64, layout="compact"):
    layout, x_remap = (layout, "auto") if isinstance(layout, str) else layout
    return argcsr.argcsr_from_csr(
        (A.num_rows, A.num_cols, A.row_pointers, A.columns, A.values.astype(dtype)), tpg, dcs, layout=layout,
        x_remap=x_remap)


def assert_same_layout(dev, ref_m: oracle.ArgCsr, where: str = "") -> None:
    assert dev.num_groups == ref_m.groups.shape[0], f"{where}: group count {dev.num_groups} != {ref_m.groups.shape[0]}"
    assert dev.total_slots == ref_m.total_slots, f"{where}: total slots"
    assert np.array_equal(dev.groups_array, ref_m.groups), f"{where}: groups differ"
    assert np.array_equal(dev.threads_mapping, ref_m.threads_mapping), f"{where}: threads_mapping differs"
    assert np.array_equal(dev.columns, ref_m.columns), f"{where}: columns differ"
    assert dev.values.tobytes() == ref_m.values.tobytes(), f"{where}: values differ"


def bits(a: np.ndarray) -> bytes:
    return np.ascontiguousarray(a, dtype=np.float64).tobytes()
