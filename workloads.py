"""Synthetic matrices of the BASELINE.json configurations (SURVEY.md §8(d),
Appendix C) -- BENCH AND TEST INPUTS, not part of the product package.

This module lives outside `paper_1203_5737_b200/` on purpose: the reference
arm of bench.py (`--impl reference`) builds its matrix here and must not map
any of the package's native libraries.  It depends on torch only.

Every generator is a pure function of its arguments and gives the SAME matrix
bit for bit on any device: randomness comes from a counter-based hash
(splitmix64's finaliser over the element index) evaluated with wrapping int64
torch arithmetic, which CPU and CUDA compute identically, and R-MAT's quadrant
choice compares integer draws with integer thresholds.  So the B200 arm
(generating on the GPU in milliseconds) and the reference arm (generating on
the host) time the same input, and tests can regenerate any config on either
side.  The arrays follow the reference CSR layout (core.hpp:31-41): int64 row
pointers (bit-identical to u64), int32 ascending columns per row, float64
values.

  C1  stencil2d5(1024)            1,048,576 rows,   5,238,784 nnz
  C2  stencil3d27(160)            4,096,000 rows, 109,215,352 nnz
  C3  rmat(24, 16)               16,777,216 rows, ~263M nnz (hash RNG: statistically
                                  equivalent to, not identical with, the survey's
                                  mt19937_64 matrix)
  C4  arrowhead()                 8,002,048 rows, 232,799,997 nnz
  C5  stencil3d27(320)           32,768,000 rows, 879,217,912 nnz
"""
from __future__ import annotations

import hashlib
from dataclasses import dataclass

import torch

_M64 = (1 << 64) - 1


def _s64(c: int) -> int:
    """An unsigned 64-bit constant as the int64 with the same bits."""
    c &= _M64
    return c - (1 << 64) if c >= 1 << 63 else c


_GOLDEN = _s64(0x9E3779B97F4A7C15)
_MUL1 = _s64(0xBF58476D1CE4E5B9)
_MUL2 = _s64(0x94D049BB133111EB)


def _srl(z: torch.Tensor, k: int) -> torch.Tensor:
    """Logical right shift of int64 bits (torch's >> is arithmetic)."""
    return (z >> k) & ((1 << (64 - k)) - 1)


def mix64(z: torch.Tensor) -> torch.Tensor:
    """splitmix64 finaliser on int64 bit patterns (wrapping multiplies)."""
    z = (z ^ _srl(z, 30)) * _MUL1
    z = (z ^ _srl(z, 27)) * _MUL2
    return z ^ _srl(z, 31)


def hash_stream(seed: int, index: torch.Tensor) -> torch.Tensor:
    """Draw `index` of stream `seed`: 64 random bits per element."""
    return mix64(index * _GOLDEN + _s64(seed * 0xD1B54A32D192ED03 + 1))


def uniform_pm1(seed: int, index: torch.Tensor) -> torch.Tensor:
    """U[-1, 1) doubles with 53 random bits: 2 * (h >> 11) * 2^-53 - 1 (exact)."""
    return _srl(hash_stream(seed, index), 11).to(torch.float64) * (2.0 ** -52) - 1.0


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

    def digest(self) -> str:
        """sha256 over the three arrays (host copies): identity of the input."""
        h = hashlib.sha256()
        for t in (self.row_pointers, self.columns, self.values):
            h.update(t.detach().cpu().contiguous().numpy().tobytes())
        return h.hexdigest()[:16]


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
        cand, valid = [], []
        for di in (-1, 0, 1):
            mi = (i + di >= 0) & (i + di < n)
            for dj in (-1, 0, 1):
                mj = mi & (j + dj >= 0) & (j + dj < n)
                for dk in (-1, 0, 1):
                    cand.append(r + (di * n + dj) * n + dk)
                    valid.append(mj & (k + dk >= 0) & (k + dk < n))
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
         abcd=(0.57, 0.19, 0.19, 0.05), chunk: int = 1 << 22) -> SynthCsr:
    """R-MAT (a,b,c,d), `scale` bisection levels per edge, no vertex
    permutation, duplicate (r, c) removed, values U(-1, 1).

    Level l of edge e uses 32 bits of hash_stream(seed, e * 16 + l // 2) (low
    half for even l, high half for odd l), compared against the integer
    thresholds round(2^32 * (a, a+b, a+b+c)): exact on every device."""
    N = 1 << scale
    E = edge_factor * N
    a, b, c, _ = abcd
    t1, t2, t3 = (round(t * (1 << 32)) for t in (a, a + b, a + b + c))
    keys = []
    for e0 in range(0, E, chunk):
        e = torch.arange(e0, min(E, e0 + chunk), device=device, dtype=torch.int64)
        r = torch.zeros_like(e)
        col = torch.zeros_like(e)
        for lp in range((scale + 1) // 2):
            h = hash_stream(seed, e * 16 + lp)
            for half in range(2):
                if 2 * lp + half >= scale:
                    break
                p = _srl(h, 32) if half else h & 0xFFFFFFFF
                bi = (p >= t2).to(torch.int64)  # quadrants (1,0) and (1,1)
                bj = (((p >= t1) & (p < t2)) | (p >= t3)).to(torch.int64)  # (0,1) and (1,1)
                r = r * 2 + bi
                col = col * 2 + bj
        keys.append(r * N + col)
        del e, r, col
    key = torch.cat(keys)
    del keys
    key = torch.unique(key)  # sorted, duplicates removed
    rows = key // N
    cols = (key % N).to(torch.int32)
    counts = torch.bincount(rows, minlength=N)
    del rows
    rp = torch.zeros(N + 1, dtype=torch.int64, device=device)
    torch.cumsum(counts, 0, out=rp[1:])
    vals = torch.empty(key.numel(), dtype=torch.float64, device=device)
    for k0 in range(0, key.numel(), chunk):
        k1 = min(key.numel(), k0 + chunk)
        vals[k0:k1] = uniform_pm1(seed + 1000, torch.arange(k0, k1, device=device, dtype=torch.int64))
    return SynthCsr(f"rmat_s{scale}_ef{edge_factor}", N, N, rp, cols, vals)


def arrowhead(short: int = 8_000_000, dense: int = 2048, dense_nnz: int = 100_000, seed: int = 7,
              device="cuda") -> SynthCsr:
    """8M short rows with 2 + (r mod 4) nnz on a diagonal band (clipped) plus
    `dense` rows of `dense_nnz` entries (c = j * floor(N / dense_nnz)) every
    floor(N / dense)-th row; values U(-1, 1) from the hash stream."""
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
    row_start = torch.repeat_interleave(rp[:-1], counts)  # row start of every element
    within = torch.arange(nnz, device=device, dtype=torch.int64) - row_start
    del row_start
    row_of = torch.repeat_interleave(r, counts)
    dense_el = is_dense[row_of]
    del row_of
    cols[dense_el] = (within[dense_el] * step).to(torch.int32)
    cols[~dense_el] = cand[valid].to(torch.int32)
    del within, dense_el, cand, valid
    vals = uniform_pm1(seed, torch.arange(nnz, device=device, dtype=torch.int64))
    return SynthCsr(f"arrowhead_{short}_{dense}x{dense_nnz}", N, N, rp, cols, vals)


def bench_input(n: int, device="cuda", dtype=torch.float64) -> torch.Tensor:
    """x[j] = 1 + 0.0625 * (j mod 13) (proj/src/bench.cpp:143-149)."""
    return (1.0 + 0.0625 * (torch.arange(n, device=device, dtype=torch.int64) % 13).to(torch.float64)).to(dtype)


CONFIGS = {
    "C1": dict(gen=lambda d: stencil2d5(1024, d), dtype="float64", desc="2D 5-point Laplacian 1024x1024, fp64"),
    "C2": dict(gen=lambda d: stencil3d27(160, d), dtype="float64", desc="3D 27-point stencil 160^3, fp64"),
    "C3": dict(gen=lambda d: rmat(24, 16, 1, d), dtype="float64", desc="R-MAT 2^24, edge factor 16, fp64"),
    "C4": dict(gen=lambda d: arrowhead(device=d), dtype="float64", desc="arrowhead 8M short + 2048x1e5 dense, fp64"),
    "C4f32": dict(gen=lambda d: arrowhead(device=d), dtype="float32",
                  desc="arrowhead 8M short + 2048x1e5 dense, fp32"),
    "C5": dict(gen=lambda d: stencil3d27(320, d), dtype="float64", desc="3D 27-point stencil 320^3, fp64"),
}
