"""Synthetic matrices of the BASELINE.json configurations (SURVEY.md §8(d),
Appendix C), generated with torch on any device (CUDA for the bench, CPU for
the reference arm).  Deterministic for a given seed and device type.

Every generator returns a `SynthCsr` whose arrays follow the reference CSR
layout (core.hpp:31-41): int64 row pointers (bit-identical to u64), int32
ascending columns per row, float64 values.

  C1  stencil2d5(1024)            1,048,576 rows,   5,238,784 nnz
  C2  stencil3d27(160)            4,096,000 rows, 109,215,352 nnz
  C3  rmat(24, 16)               16,777,216 rows, ~263M nnz (counter-based RNG:
                                  statistically equivalent to, not identical with,
                                  the survey's mt19937_64 matrix)
  C4  arrowhead()                 8,002,048 rows, 232,799,997 nnz
  C5  stencil3d27(320)           32,768,000 rows, 879,217,912 nnz
"""
from __future__ import annotations

from dataclasses import dataclass

import torch


@dataclass
class SynthCsr:
    name: str
    num_rows: int
    num_cols: int
    row_pointers: torch.Tensor  # int64 [num_rows + 1]
    columns: torch.Tensor  # int32 [nnz]
    values: torch.Tensor  # float64 [nnz]

    @property
    def nnz(self) -> int:
        return int(self.columns.numel())

    def to(self, device) -> "SynthCsr":
        return SynthCsr(self.name, self.num_rows, self.num_cols, self.row_pointers.to(device),
                        self.columns.to(device), self.values.to(device))

    def slice_rows(self, r0: int, r1: int) -> "SynthCsr":
        """Rows [r0, r1) with row pointers rebased to 0 and all columns kept."""
        a, b = int(self.row_pointers[r0]), int(self.row_pointers[r1])
        return SynthCsr(f"{self.name}[{r0}:{r1}]", r1 - r0, self.num_cols, self.row_pointers[r0:r1 + 1] - a,
                        self.columns[a:b], self.values[a:b])


def _from_candidates(name: str, n_rows: int, n_cols: int, cand: torch.Tensor, valid: torch.Tensor,
                     vals: torch.Tensor) -> SynthCsr:
    counts = valid.sum(dim=1)
    rp = torch.zeros(n_rows + 1, dtype=torch.int64, device=cand.device)
    torch.cumsum(counts, 0, out=rp[1:])
    return SynthCsr(name, n_rows, n_cols, rp, cand[valid].to(torch.int32), vals[valid])


def stencil2d5(n: int = 1024, device="cuda") -> SynthCsr:
    """5-point Laplacian, r = i*n + j, diag 4, neighbours -1, ascending columns."""
    N = n * n
    r = torch.arange(N, device=device, dtype=torch.int64)
    i, j = r // n, r % n
    offs = [(-n, i > 0), (-1, j > 0), (0, torch.ones_like(i, dtype=torch.bool)), (1, j < n - 1), (n, i < n - 1)]
    cand = torch.stack([r + o for o, _ in offs], dim=1)
    valid = torch.stack([m for _, m in offs], dim=1)
    vals = torch.full(cand.shape, -1.0, dtype=torch.float64, device=device)
    vals[:, 2] = 4.0
    return _from_candidates(f"stencil2d5_{n}", N, N, cand, valid, vals)


def stencil3d27(n: int = 160, device="cuda", row_chunk: int = 1 << 22) -> SynthCsr:
    """27-point stencil, r = (i*n + j)*n + k, diag 26, neighbours -1; the
    di -> dj -> dk nesting yields ascending columns.  Built in row chunks to
    bound temporary memory at n = 320."""
    N = n ** 3
    rps, cols, vals = [torch.zeros(1, dtype=torch.int64, device=device)], [], []
    base = 0
    for r0 in range(0, N, row_chunk):
        r = torch.arange(r0, min(N, r0 + row_chunk), device=device, dtype=torch.int64)
        i, j, k = r // (n * n), (r // n) % n, r % n
        cand, valid, v = [], [], []
        for di in (-1, 0, 1):
            mi = (i + di >= 0) & (i + di < n)
            for dj in (-1, 0, 1):
                mj = mi & (j + dj >= 0) & (j + dj < n)
                for dk in (-1, 0, 1):
                    m = mj & (k + dk >= 0) & (k + dk < n)
                    cand.append(r + (di * n + dj) * n + dk)
                    valid.append(m)
        cand = torch.stack(cand, 1)
        valid = torch.stack(valid, 1)
        vv = torch.full(cand.shape, -1.0, dtype=torch.float64, device=device)
        vv[:, 13] = 26.0
        counts = valid.sum(1)
        rps.append(torch.cumsum(counts, 0) + base)
        base += int(counts.sum())
        cols.append(cand[valid].to(torch.int32))
        vals.append(vv[valid])
        del cand, valid, vv
    return SynthCsr(f"stencil3d27_{n}", N, N, torch.cat(rps), torch.cat(cols), torch.cat(vals))


def rmat(scale: int = 24, edge_factor: int = 16, seed: int = 1, device="cuda",
         abcd=(0.57, 0.19, 0.19, 0.05), chunk: int = 1 << 24) -> SynthCsr:
    """R-MAT (a,b,c,d), `scale` bisection levels per edge, no vertex
    permutation, duplicate (r, c) removed, values U(-1, 1)."""
    N = 1 << scale
    E = edge_factor * N
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    a, b, c, _ = abcd
    t1, t2, t3 = a, a + b, a + b + c
    keys = []
    for e0 in range(0, E, chunk):
        m = min(chunk, E - e0)
        r = torch.zeros(m, dtype=torch.int64, device=device)
        col = torch.zeros(m, dtype=torch.int64, device=device)
        for _ in range(scale):
            p = torch.rand(m, generator=g, device=device, dtype=torch.float64)
            bi = (p >= t2).to(torch.int64)  # quadrants (1,0) and (1,1)
            bj = ((p >= t1) & (p < t2) | (p >= t3)).to(torch.int64)  # (0,1) and (1,1)
            r = r * 2 + bi
            col = col * 2 + bj
        keys.append(r * N + col)
    key = torch.unique(torch.cat(keys))  # sorted
    rows = key // N
    cols = (key % N).to(torch.int32)
    counts = torch.bincount(rows, minlength=N)
    rp = torch.zeros(N + 1, dtype=torch.int64, device=device)
    torch.cumsum(counts, 0, out=rp[1:])
    vals = torch.rand(key.numel(), generator=g, device=device, dtype=torch.float64) * 2.0 - 1.0
    return SynthCsr(f"rmat_s{scale}_ef{edge_factor}", N, N, rp, cols, vals)


def arrowhead(short: int = 8_000_000, dense: int = 2048, dense_nnz: int = 100_000, seed: int = 7,
              device="cuda") -> SynthCsr:
    """8M short rows with 2 + (r mod 4) nnz on a diagonal band (clipped) plus
    `dense` rows of `dense_nnz` entries (c = j * floor(N / dense_nnz)) every
    floor(N / dense)-th row; values U(-1, 1)."""
    N = short + dense
    stride, step = N // dense, N // dense_nnz
    r = torch.arange(N, device=device, dtype=torch.int64)
    is_dense = (r % stride == stride - 1) & (r // stride < dense)
    kk = 2 + r % 4
    j = torch.arange(5, device=device, dtype=torch.int64)
    cand = r[:, None] - (kk // 2)[:, None] + j[None, :]
    valid = (j[None, :] < kk[:, None]) & (cand >= 0) & (cand < N) & ~is_dense[:, None]
    counts = torch.where(is_dense, torch.full_like(r, dense_nnz), valid.sum(1))
    rp = torch.zeros(N + 1, dtype=torch.int64, device=device)
    torch.cumsum(counts, 0, out=rp[1:])
    nnz = int(rp[-1])
    cols = torch.empty(nnz, dtype=torch.int32, device=device)
    short_pos = torch.repeat_interleave(rp[:-1], counts)  # row start of every element
    within = torch.arange(nnz, device=device, dtype=torch.int64) - short_pos
    row_of = torch.repeat_interleave(r, counts)
    dense_el = is_dense[row_of]
    cols[dense_el] = (within[dense_el] * step).to(torch.int32)
    cols[~dense_el] = cand[valid].to(torch.int32)
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    vals = torch.rand(nnz, generator=g, device=device, dtype=torch.float64) * 2.0 - 1.0
    return SynthCsr(f"arrowhead_{short}_{dense}x{dense_nnz}", N, N, rp, cols, vals)


def bench_input(n: int, device="cuda", dtype=torch.float64) -> torch.Tensor:
    """x[j] = 1 + 0.0625 * (j mod 13) (proj/src/bench.cpp:143-149)."""
    return (1.0 + 0.0625 * (torch.arange(n, device=device, dtype=torch.int64) % 13).to(torch.float64)).to(dtype)


CONFIGS = {
    "C1": dict(gen=lambda d: stencil2d5(1024, d), dtype="float64", desc="2D 5-point Laplacian 1024x1024, fp64"),
    "C2": dict(gen=lambda d: stencil3d27(160, d), dtype="float64", desc="3D 27-point stencil 160^3, fp64"),
    "C3": dict(gen=lambda d: rmat(24, 16, 1, d), dtype="float64", desc="R-MAT 2^24, edge factor 16, fp64"),
    "C4": dict(gen=lambda d: arrowhead(device=d), dtype="float64", desc="arrowhead 8M short + 2048x1e5 dense, fp64"),
    "C4f32": dict(gen=lambda d: arrowhead(device=d), dtype="float32", desc="arrowhead 8M short + 2048x1e5 dense, fp32"),
    "C5": dict(gen=lambda d: stencil3d27(320, d), dtype="float64", desc="3D 27-point stencil 320^3, fp64"),
}
