"""TEST INFRASTRUCTURE ONLY — the CPU checkers for the ARG-CSR hot path.

Two ctypes front-ends:

* ``orc`` — liboracle.so, the plain-C restatement (argcsr_oracle.c) of the
  reference algorithm (proj/src/argcsr.cpp, core.cpp, bench.cpp).
* ``ref`` — _ref/libargcsr_ref.so, the UNMODIFIED reference library compiled
  from /root/reference/proj/src/*.cpp plus ref_shim.cpp (see Makefile).  It
  pins ``orc``, generates the reference test corpus (proj/tests/support.hpp),
  and is the timed CPU baseline.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs may import this package, and only as the checker.  The product path
(paper_1203_5737_b200) never imports it.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_SO = HERE / "liboracle.so"
REF_SO = HERE / "_ref" / "libargcsr_ref.so"

u64p = C.POINTER(C.c_uint64)
i32p = C.POINTER(C.c_int32)
f64p = C.POINTER(C.c_double)


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


@dataclass
class Csr:
    """A CSR matrix as numpy arrays (core.hpp:31-41 fields)."""

    num_rows: int
    num_cols: int
    row_pointers: np.ndarray  # u64 [num_rows+1]
    columns: np.ndarray  # i32 [nnz]
    values: np.ndarray  # f64 [nnz]

    @property
    def nnz(self) -> int:
        return int(self.values.size)


@dataclass
class ArgCsr:
    """The reference ArgCsrMatrix layout (argcsr.hpp:52-63) as numpy arrays."""

    num_rows: int
    num_cols: int
    threads_per_group: int
    groups: np.ndarray  # u64 [G, 4]: first_row, size, offset, chunk_size
    threads_mapping: np.ndarray  # u64 [num_rows]
    values: np.ndarray  # f64 [total_slots]
    columns: np.ndarray  # i32 [total_slots]

    @property
    def total_slots(self) -> int:
        return int(self.values.size)


def _p(a: np.ndarray, t):
    return a.ctypes.data_as(t)


def _csr_arrays(A: Csr):
    rp = np.ascontiguousarray(A.row_pointers, dtype=np.uint64)
    cols = np.ascontiguousarray(A.columns, dtype=np.int32)
    vals = np.ascontiguousarray(A.values, dtype=np.float64)
    return rp, cols, vals


class _Orc:
    def __init__(self, path: Path = ORACLE_SO):
        self.lib = C.CDLL(str(path))
        L = self.lib
        L.orc_last_error.restype = C.c_char_p
        L.orc_argcsr_sizes.argtypes = [C.c_uint64, u64p, C.c_uint64, C.c_uint64, u64p, u64p]
        L.orc_argcsr_from_csr.argtypes = [C.c_uint64, u64p, i32p, f64p, C.c_uint64, C.c_uint64, u64p, u64p, f64p, i32p]
        L.orc_partition_groups.argtypes = [u64p, C.c_uint64, C.c_uint64, C.c_uint64, u64p, u64p]
        L.orc_assign_threads.argtypes = [u64p, C.c_uint64, C.c_uint64, u64p, u64p, u64p, u64p]
        L.orc_spmv_argcsr.argtypes = [C.c_uint64] * 4 + [u64p, u64p, f64p, i32p, f64p, C.c_uint64, f64p]
        L.orc_spmv_argcsr_parallel.argtypes = [C.c_uint64] * 4 + [u64p, u64p, f64p, i32p, f64p, C.c_uint64, f64p,
                                                                   C.c_uint64]
        L.orc_spmv_argcsr_groups.argtypes = [C.c_uint64, u64p, u64p, f64p, i32p, f64p, C.c_uint64, C.c_uint64, f64p]
        L.orc_csr_from_argcsr_rp.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, u64p, u64p, i32p, u64p]
        L.orc_csr_from_argcsr.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, u64p, u64p, f64p, i32p, u64p, i32p, f64p]
        L.orc_spmv_csr.argtypes = [C.c_uint64, C.c_uint64, u64p, i32p, f64p, f64p, C.c_uint64, f64p]
        L.orc_abs_row_sums.argtypes = [C.c_uint64, u64p, i32p, f64p, f64p, f64p]
        L.orc_padding_stats.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, u64p, u64p, C.c_uint64, i32p, u64p, u64p,
                                        u64p]

    def _check(self, st: int):
        if st:
            raise OracleError(st, self.lib.orc_last_error().decode())

    def partition_groups(self, counts, tpg: int, dcs: int) -> np.ndarray:
        c = np.ascontiguousarray(counts, dtype=np.uint64)
        out = np.zeros(2 * max(c.size, 1), dtype=np.uint64)
        n = C.c_uint64(0)
        self._check(self.lib.orc_partition_groups(_p(c, u64p), c.size, tpg, dcs, _p(out, u64p), C.byref(n)))
        return out[: 2 * n.value].reshape(-1, 2)

    def assign_threads(self, counts, tpg: int):
        c = np.ascontiguousarray(counts, dtype=np.uint64)
        tpr = np.zeros(max(c.size, 1), dtype=np.uint64)
        ch, asg, fr = C.c_uint64(), C.c_uint64(), C.c_uint64()
        self._check(self.lib.orc_assign_threads(_p(c, u64p), c.size, tpg, _p(tpr, u64p), C.byref(ch), C.byref(asg),
                                                C.byref(fr)))
        return tpr[: c.size], ch.value, asg.value, fr.value

    def argcsr_from_csr(self, A: Csr, tpg: int = 128, dcs: int = 1) -> ArgCsr:
        rp, cols, vals = _csr_arrays(A)
        G, S = C.c_uint64(), C.c_uint64()
        self._check(self.lib.orc_argcsr_sizes(A.num_rows, _p(rp, u64p), tpg, dcs, C.byref(G), C.byref(S)))
        g4 = np.zeros((G.value, 4), dtype=np.uint64)
        tm = np.zeros(A.num_rows, dtype=np.uint64)
        ov = np.zeros(S.value, dtype=np.float64)
        oc = np.zeros(S.value, dtype=np.int32)
        self._check(self.lib.orc_argcsr_from_csr(A.num_rows, _p(rp, u64p), _p(cols, i32p), _p(vals, f64p), tpg, dcs,
                                                 _p(g4, u64p), _p(tm, u64p), _p(ov, f64p), _p(oc, i32p)))
        return ArgCsr(A.num_rows, A.num_cols, tpg, g4, tm, ov, oc)

    def spmv_argcsr(self, M: ArgCsr, x) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.zeros(M.num_rows, dtype=np.float64)
        g4 = np.ascontiguousarray(M.groups, dtype=np.uint64)
        self._check(self.lib.orc_spmv_argcsr(M.num_rows, M.num_cols, M.threads_per_group, g4.shape[0], _p(g4, u64p),
                                             _p(M.threads_mapping, u64p), _p(M.values, f64p), _p(M.columns, i32p),
                                             _p(x, f64p), x.size, _p(y, f64p)))
        return y

    def spmv_argcsr_parallel(self, M: ArgCsr, x, workers: int) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.zeros(M.num_rows, dtype=np.float64)
        g4 = np.ascontiguousarray(M.groups, dtype=np.uint64)
        self._check(self.lib.orc_spmv_argcsr_parallel(M.num_rows, M.num_cols, M.threads_per_group, g4.shape[0],
                                                      _p(g4, u64p), _p(M.threads_mapping, u64p), _p(M.values, f64p),
                                                      _p(M.columns, i32p), _p(x, f64p), x.size, _p(y, f64p), workers))
        return y

    def spmv_csr(self, A: Csr, x) -> np.ndarray:
        rp, cols, vals = _csr_arrays(A)
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.zeros(A.num_rows, dtype=np.float64)
        self._check(self.lib.orc_spmv_csr(A.num_rows, A.num_cols, _p(rp, u64p), _p(cols, i32p), _p(vals, f64p),
                                          _p(x, f64p), x.size, _p(y, f64p)))
        return y

    def abs_row_sums(self, A: Csr, x) -> np.ndarray:
        rp, cols, vals = _csr_arrays(A)
        x = np.ascontiguousarray(x, dtype=np.float64)
        out = np.zeros(A.num_rows, dtype=np.float64)
        self.lib.orc_abs_row_sums(A.num_rows, _p(rp, u64p), _p(cols, i32p), _p(vals, f64p), _p(x, f64p),
                                  _p(out, f64p))
        return out

    def csr_from_argcsr(self, M: ArgCsr) -> Csr:
        g4 = np.ascontiguousarray(M.groups, dtype=np.uint64)
        rp = np.zeros(M.num_rows + 1, dtype=np.uint64)
        self._check(self.lib.orc_csr_from_argcsr_rp(M.num_rows, M.threads_per_group, g4.shape[0], _p(g4, u64p),
                                                    _p(M.threads_mapping, u64p), _p(M.columns, i32p), _p(rp, u64p)))
        nnz = int(rp[-1])
        oc = np.zeros(nnz, dtype=np.int32)
        ov = np.zeros(nnz, dtype=np.float64)
        self._check(self.lib.orc_csr_from_argcsr(M.num_rows, M.threads_per_group, g4.shape[0], _p(g4, u64p),
                                                 _p(M.threads_mapping, u64p), _p(M.values, f64p), _p(M.columns, i32p),
                                                 _p(rp, u64p), _p(oc, i32p), _p(ov, f64p)))
        return Csr(M.num_rows, M.num_cols, rp, oc, ov)

    def padding_stats(self, M: ArgCsr):
        g4 = np.ascontiguousarray(M.groups, dtype=np.uint64)
        e, p, t = C.c_uint64(), C.c_uint64(), C.c_uint64()
        self.lib.orc_padding_stats(M.num_rows, M.threads_per_group, g4.shape[0], _p(g4, u64p),
                                   _p(M.threads_mapping, u64p), M.total_slots, _p(M.columns, i32p), C.byref(e),
                                   C.byref(p), C.byref(t))
        return e.value, p.value, t.value


class _Ref:
    """The compiled reference library (test/baseline only)."""

    def __init__(self, path: Path = REF_SO):
        self.lib = C.CDLL(str(path))
        L = self.lib
        vp = C.c_void_p
        L.ref_last_error.restype = C.c_char_p
        L.ref_csr_new.restype = vp
        L.ref_csr_new.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, u64p, i32p, f64p]
        L.ref_csr_from_triplets.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, u64p, u64p, f64p, C.POINTER(vp)]
        L.ref_csr_shape.argtypes = [vp, u64p, u64p, u64p]
        L.ref_csr_copy.argtypes = [vp, u64p, i32p, f64p]
        L.ref_csr_free.argtypes = [vp]
        for f in ("ref_fixture_e8",):
            getattr(L, f).restype = vp
        L.ref_fixture_skew.restype = vp
        L.ref_fixture_skew.argtypes = [C.c_uint64]
        L.ref_fixture_uniform.restype = vp
        L.ref_fixture_uniform.argtypes = [C.c_uint64] * 3
        L.ref_probe_vector.argtypes = [C.c_uint64, C.c_uint32, f64p]
        L.ref_corpus_new.restype = vp
        L.ref_corpus_new.argtypes = [C.c_uint64, C.c_uint32]
        L.ref_corpus_size.restype = C.c_uint64
        L.ref_corpus_size.argtypes = [vp]
        L.ref_corpus_get.restype = vp
        L.ref_corpus_get.argtypes = [vp, C.c_uint64]
        L.ref_corpus_free.argtypes = [vp]
        L.ref_partition_groups.argtypes = [u64p, C.c_uint64, C.c_uint64, C.c_uint64, u64p, u64p]
        L.ref_assign_threads.argtypes = [u64p, C.c_uint64, C.c_uint64, u64p, u64p, u64p, u64p]
        L.ref_argcsr_from_csr.argtypes = [vp, C.c_uint64, C.c_uint64, C.POINTER(vp)]
        L.ref_argcsr_info.argtypes = [vp, u64p, u64p, u64p, u64p, u64p]
        L.ref_argcsr_export.argtypes = [vp, u64p, u64p, f64p, i32p]
        L.ref_argcsr_import.restype = vp
        L.ref_argcsr_import.argtypes = [C.c_uint64] * 4 + [u64p, u64p, C.c_uint64, f64p, i32p]
        L.ref_argcsr_free.argtypes = [vp]
        L.ref_csr_from_argcsr.argtypes = [vp, C.POINTER(vp)]
        L.ref_chunk_entries.argtypes = [vp, C.c_uint64, C.c_uint64, f64p, i32p, u64p]
        L.ref_padding_stats.argtypes = [vp, u64p, u64p, u64p, f64p, u64p]
        L.ref_balance_stats.argtypes = [vp, u64p, f64p, f64p]
        L.ref_spmv_argcsr.argtypes = [vp, f64p, C.c_uint64, f64p]
        L.ref_spmv_csr.argtypes = [vp, f64p, C.c_uint64, f64p]
        L.ref_time_spmv_argcsr_parallel.argtypes = [vp, f64p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, f64p,
                                                    f64p]
        L.ref_time_spmv_csr_parallel.argtypes = [vp, f64p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, f64p]
        L.ref_write_binary_argcsr.argtypes = [vp, C.c_char_p]
        L.ref_write_binary_csr.argtypes = [vp, C.c_char_p]
        L.ref_ellpack_from_csr.restype = vp
        L.ref_ellpack_from_csr.argtypes = [vp]
        L.ref_sliced_from_csr.argtypes = [vp, C.c_uint64, C.POINTER(vp)]
        L.ref_ell_fields.argtypes = [vp, u64p, u64p, f64p, i32p]
        L.ref_sell_fields.argtypes = [vp, u64p, u64p, u64p, u64p, f64p, i32p]
        L.ref_spmv_ellpack.argtypes = [vp, f64p, C.c_uint64, f64p]
        L.ref_spmv_sliced.argtypes = [vp, f64p, C.c_uint64, f64p]
        L.ref_ell_free.argtypes = [vp]
        L.ref_sell_free.argtypes = [vp]
        L.ref_hardware_threads.restype = C.c_uint64

    def _check(self, st: int):
        if st:
            raise OracleError(st, self.lib.ref_last_error().decode())

    # ------------------------------------------------------------ CSR helpers
    def _csr_from_handle(self, h) -> Csr:
        nr, nc, nnz = C.c_uint64(), C.c_uint64(), C.c_uint64()
        self.lib.ref_csr_shape(h, C.byref(nr), C.byref(nc), C.byref(nnz))
        rp = np.zeros(nr.value + 1, dtype=np.uint64)
        cols = np.zeros(nnz.value, dtype=np.int32)
        vals = np.zeros(nnz.value, dtype=np.float64)
        self.lib.ref_csr_copy(h, _p(rp, u64p), _p(cols, i32p), _p(vals, f64p))
        return Csr(nr.value, nc.value, rp, cols, vals)

    def _take(self, h) -> Csr:
        try:
            return self._csr_from_handle(h)
        finally:
            self.lib.ref_csr_free(h)

    def csr_handle(self, A: Csr):
        rp, cols, vals = _csr_arrays(A)
        return self.lib.ref_csr_new(A.num_rows, A.num_cols, A.nnz, _p(rp, u64p), _p(cols, i32p), _p(vals, f64p))

    def csr_from_triplets(self, num_rows: int, num_cols: int, entries) -> Csr:
        rows = np.array([e[0] for e in entries], dtype=np.uint64)
        cols = np.array([e[1] for e in entries], dtype=np.uint64)
        vals = np.array([e[2] for e in entries], dtype=np.float64)
        h = C.c_void_p()
        self._check(self.lib.ref_csr_from_triplets(num_rows, num_cols, len(entries), _p(rows, u64p), _p(cols, u64p),
                                                   _p(vals, f64p), C.byref(h)))
        return self._take(h)

    def e8(self) -> Csr:
        return self._take(self.lib.ref_fixture_e8())

    def skew(self, k: int) -> Csr:
        return self._take(self.lib.ref_fixture_skew(k))

    def uniform(self, rows: int, cols: int, per_row: int) -> Csr:
        return self._take(self.lib.ref_fixture_uniform(rows, cols, per_row))

    def probe_vector(self, n: int, salt: int = 0) -> np.ndarray:
        x = np.zeros(n, dtype=np.float64)
        self.lib.ref_probe_vector(n, salt, _p(x, f64p))
        return x

    def corpus(self, count: int, seed: int = 20260822) -> list[Csr]:
        h = self.lib.ref_corpus_new(count, seed)
        try:
            return [self._csr_from_handle(self.lib.ref_corpus_get(h, i)) for i in range(self.lib.ref_corpus_size(h))]
        finally:
            self.lib.ref_corpus_free(h)

    # ------------------------------------------------------------- the path
    def partition_groups(self, counts, tpg: int, dcs: int) -> np.ndarray:
        c = np.ascontiguousarray(counts, dtype=np.uint64)
        out = np.zeros(2 * max(c.size, 1), dtype=np.uint64)
        n = C.c_uint64(0)
        self._check(self.lib.ref_partition_groups(_p(c, u64p), c.size, tpg, dcs, _p(out, u64p), C.byref(n)))
        return out[: 2 * n.value].reshape(-1, 2)

    def assign_threads(self, counts, tpg: int):
        c = np.ascontiguousarray(counts, dtype=np.uint64)
        tpr = np.zeros(max(c.size, 1), dtype=np.uint64)
        ch, asg, fr = C.c_uint64(), C.c_uint64(), C.c_uint64()
        self._check(self.lib.ref_assign_threads(_p(c, u64p), c.size, tpg, _p(tpr, u64p), C.byref(ch), C.byref(asg),
                                                C.byref(fr)))
        return tpr[: c.size], ch.value, asg.value, fr.value

    def argcsr_handle(self, A: Csr, tpg: int = 128, dcs: int = 1):
        """Reference-converted ArgCsrMatrix handle (caller frees with free_argcsr)."""
        hc = self.csr_handle(A)
        try:
            h = C.c_void_p()
            self._check(self.lib.ref_argcsr_from_csr(hc, tpg, dcs, C.byref(h)))
            return h
        finally:
            self.lib.ref_csr_free(hc)

    def export(self, h) -> ArgCsr:
        nr, nc, t, G, S = (C.c_uint64() for _ in range(5))
        self.lib.ref_argcsr_info(h, C.byref(nr), C.byref(nc), C.byref(t), C.byref(G), C.byref(S))
        g4 = np.zeros((G.value, 4), dtype=np.uint64)
        tm = np.zeros(nr.value, dtype=np.uint64)
        v = np.zeros(S.value, dtype=np.float64)
        c = np.zeros(S.value, dtype=np.int32)
        self.lib.ref_argcsr_export(h, _p(g4, u64p), _p(tm, u64p), _p(v, f64p), _p(c, i32p))
        return ArgCsr(nr.value, nc.value, t.value, g4, tm, v, c)

    def argcsr_from_csr(self, A: Csr, tpg: int = 128, dcs: int = 1) -> ArgCsr:
        h = self.argcsr_handle(A, tpg, dcs)
        try:
            return self.export(h)
        finally:
            self.lib.ref_argcsr_free(h)

    def import_argcsr(self, M: ArgCsr):
        g4 = np.ascontiguousarray(M.groups, dtype=np.uint64)
        tm = np.ascontiguousarray(M.threads_mapping, dtype=np.uint64)
        v = np.ascontiguousarray(M.values, dtype=np.float64)
        c = np.ascontiguousarray(M.columns, dtype=np.int32)
        return self.lib.ref_argcsr_import(M.num_rows, M.num_cols, M.threads_per_group, g4.shape[0], _p(g4, u64p),
                                          _p(tm, u64p), v.size, _p(v, f64p), _p(c, i32p))

    def free_argcsr(self, h):
        self.lib.ref_argcsr_free(h)

    def spmv_argcsr_h(self, h, x, num_rows: int) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.zeros(num_rows, dtype=np.float64)
        self._check(self.lib.ref_spmv_argcsr(h, _p(x, f64p), x.size, _p(y, f64p)))
        return y

    def spmv_argcsr(self, M: ArgCsr, x) -> np.ndarray:
        h = self.import_argcsr(M)
        try:
            return self.spmv_argcsr_h(h, x, M.num_rows)
        finally:
            self.lib.ref_argcsr_free(h)

    def spmv_csr(self, A: Csr, x) -> np.ndarray:
        h = self.csr_handle(A)
        try:
            x = np.ascontiguousarray(x, dtype=np.float64)
            y = np.zeros(A.num_rows, dtype=np.float64)
            self._check(self.lib.ref_spmv_csr(h, _p(x, f64p), x.size, _p(y, f64p)))
            return y
        finally:
            self.lib.ref_csr_free(h)

    def csr_from_argcsr(self, M: ArgCsr) -> Csr:
        h = self.import_argcsr(M)
        try:
            out = C.c_void_p()
            self._check(self.lib.ref_csr_from_argcsr(h, C.byref(out)))
            return self._take(out)
        finally:
            self.lib.ref_argcsr_free(h)

    def chunk_entries(self, M: ArgCsr, g: int, c: int):
        h = self.import_argcsr(M)
        try:
            cap = int(M.groups[:, 3].max()) + 1 if M.groups.size else 1
            v = np.zeros(cap, dtype=np.float64)
            cc = np.zeros(cap, dtype=np.int32)
            n = C.c_uint64()
            self._check(self.lib.ref_chunk_entries(h, g, c, _p(v, f64p), _p(cc, i32p), C.byref(n)))
            return [(float(v[i]), int(cc[i])) for i in range(n.value)]
        finally:
            self.lib.ref_argcsr_free(h)

    def padding_stats(self, M: ArgCsr):
        h = self.import_argcsr(M)
        try:
            e, p, t, b = C.c_uint64(), C.c_uint64(), C.c_uint64(), C.c_uint64()
            r = C.c_double()
            self._check(self.lib.ref_padding_stats(h, C.byref(e), C.byref(p), C.byref(t), C.byref(r), C.byref(b)))
            return dict(explicit_nnz=e.value, assigned_padded_slots=p.value, total_allocated_slots=t.value,
                        padding_ratio=r.value, estimated_bytes=b.value)
        finally:
            self.lib.ref_argcsr_free(h)

    def balance_stats(self, M: ArgCsr):
        """balance_stats(const ArgCsrMatrix&) of the compiled reference (analysis.cpp:198-208)."""
        h = self.import_argcsr(M)
        try:
            per = np.zeros(M.groups.shape[0], dtype=np.uint64)
            mom, cv = C.c_double(), C.c_double()
            self._check(self.lib.ref_balance_stats(h, _p(per, u64p), C.byref(mom), C.byref(cv)))
            return per, mom.value, cv.value
        finally:
            self.lib.ref_argcsr_free(h)

    def time_spmv_argcsr_parallel(self, h, x, workers: int, warmup: int, iters: int, num_rows: int):
        x = np.ascontiguousarray(x, dtype=np.float64)
        times = np.zeros(iters, dtype=np.float64)
        y = np.zeros(num_rows, dtype=np.float64)
        self._check(self.lib.ref_time_spmv_argcsr_parallel(h, _p(x, f64p), x.size, workers, warmup, iters,
                                                           _p(times, f64p), _p(y, f64p)))
        return times, y

    def write_binary(self, M: ArgCsr, path: str):
        h = self.import_argcsr(M)
        try:
            self._check(self.lib.ref_write_binary_argcsr(h, path.encode()))
        finally:
            self.lib.ref_argcsr_free(h)

    def read_matrix_market(self, path: str) -> Csr:
        """The reference's read_matrix_market_file, run in a helper process
        (_ref/ref_mm_tool) that writes the CsrMatrix as the reference's CSR
        container; parsed here (io.cpp:250-257, 313-320)."""
        import struct
        import subprocess
        import tempfile

        with tempfile.TemporaryDirectory() as d:
            out = Path(d) / "a.spfmt"
            r = subprocess.run([str(REF_SO.parent / "ref_mm_tool"), str(path), str(out)], capture_output=True,
                               text=True)
            if r.returncode:
                raise OracleError(-1, r.stdout.strip() or r.stderr.strip())
            raw = out.read_bytes()
        assert raw[:8] == b"SPFMTBIN" and raw[12] == 0
        nr, nc = struct.unpack_from("<2Q", raw, 13)
        pos, arrs = 29, []
        for dt in ("<f8", "<i4", "<u8"):
            (n,) = struct.unpack_from("<Q", raw, pos)
            arrs.append(np.frombuffer(raw, dt, n, pos + 8).copy())
            pos += 8 + n * np.dtype(dt).itemsize
        vals, cols, rp = arrs
        return Csr(nr, nc, rp, cols, vals)

    def ellpack(self, A: Csr, x=None):
        """ellpack_from_csr(A) fields (width, values, columns) and, with x, spmv_ellpack(M, x)."""
        h = self.csr_handle(A)
        e = self.lib.ref_ellpack_from_csr(h)
        self.lib.ref_csr_free(h)
        try:
            w, n = C.c_uint64(), C.c_uint64()
            self.lib.ref_ell_fields(e, C.byref(w), C.byref(n), None, None)
            vals, cols = np.zeros(n.value), np.zeros(n.value, np.int32)
            self.lib.ref_ell_fields(e, C.byref(w), C.byref(n), _p(vals, f64p), _p(cols, i32p))
            y = None
            if x is not None:
                x = np.ascontiguousarray(x, np.float64)
                y = np.zeros(A.num_rows)
                self._check(self.lib.ref_spmv_ellpack(e, _p(x, f64p), x.size, _p(y, f64p)))
            return w.value, vals, cols, y
        finally:
            self.lib.ref_ell_free(e)

    def sliced(self, A: Csr, slice_size: int, x=None):
        """sliced_from_csr(A, slice_size) fields and, with x, spmv_sliced(M, x)."""
        h = self.csr_handle(A)
        out = C.c_void_p()
        st = self.lib.ref_sliced_from_csr(h, slice_size, C.byref(out))
        self.lib.ref_csr_free(h)
        self._check(st)
        e = out.value
        try:
            ns, n = C.c_uint64(), C.c_uint64()
            self.lib.ref_sell_fields(e, C.byref(ns), C.byref(n), None, None, None, None)
            w, o = np.zeros(ns.value, np.uint64), np.zeros(ns.value, np.uint64)
            vals, cols = np.zeros(n.value), np.zeros(n.value, np.int32)
            self.lib.ref_sell_fields(e, C.byref(ns), C.byref(n), _p(w, u64p), _p(o, u64p), _p(vals, f64p),
                                     _p(cols, i32p))
            y = None
            if x is not None:
                x = np.ascontiguousarray(x, np.float64)
                y = np.zeros(A.num_rows)
                self._check(self.lib.ref_spmv_sliced(e, _p(x, f64p), x.size, _p(y, f64p)))
            return w, o, vals, cols, y
        finally:
            self.lib.ref_sell_free(e)

    def write_binary_csr(self, A: Csr, path: str):
        h = self.csr_handle(A)
        try:
            self._check(self.lib.ref_write_binary_csr(h, path.encode()))
        finally:
            self.lib.ref_csr_free(h)

    def hardware_threads(self) -> int:
        return int(self.lib.ref_hardware_threads())


_orc = None
_ref = None


def orc() -> _Orc:
    global _orc
    if _orc is None:
        _orc = _Orc()
    return _orc


def ref_available() -> bool:
    return REF_SO.exists()


def ref() -> _Ref:
    global _ref
    if _ref is None:
        _ref = _Ref()
    return _ref


def bench_input(n: int) -> np.ndarray:
    """x[j] = 1 + 0.0625 * (j mod 13) (proj/src/bench.cpp:143-149)."""
    return 1.0 + 0.0625 * (np.arange(n, dtype=np.uint64) % 13).astype(np.float64)


def build() -> None:
    """Compile liboracle.so and, when /root/reference is present, _ref/."""
    import subprocess

    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
