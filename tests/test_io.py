"""The reference's binary container (SPFMTBIN, proj/src/io.cpp:17-22, 242-366)
on the device path: write_binary of a device handle is byte-identical to the
reference's file, read_binary imports it (or converts a CSR container), and
corrupted streams fail like proj/tests/test_io.cpp:163-190.

The golden containers under tests/golden/ were written by the compiled
reference (tests/golden/make_golden.py)."""
import struct
from pathlib import Path

import numpy as np
import pytest

from helpers import LAYOUTS, assert_same_layout, bits, powerlaw_csr, to_dev

GOLDEN = Path(__file__).resolve().parent / "golden"


def parse_argcsr_container(raw: bytes):
    """A plain restatement of read_binary's ARG-CSR branch (io.cpp:343-363)."""
    assert raw[:8] == b"SPFMTBIN"
    version, tag = struct.unpack_from("<IB", raw, 8)
    assert (version, tag) == (1, 3)
    pos = 13
    rows, cols, tpg, G = struct.unpack_from("<4Q", raw, pos)
    pos += 32
    groups = np.frombuffer(raw, "<u8", 4 * G, pos).reshape(G, 4)
    pos += 32 * G
    out = []
    for dt in ("<u8", "<f8", "<i4"):
        (n,) = struct.unpack_from("<Q", raw, pos)
        pos += 8
        out.append(np.frombuffer(raw, dt, n, pos))
        pos += n * np.dtype(dt).itemsize
    assert pos == len(raw)
    return rows, cols, tpg, groups, *out


# ------------------------------------------------------------------ CPU only
def test_golden_container_matches_golden_arrays():
    """The container layout we write is the one the reference wrote."""
    rows, cols, tpg, groups, tm, vals, columns = parse_argcsr_container(
        (GOLDEN / "e8_argcsr_12_2.spfmt").read_bytes())
    e8 = np.load(GOLDEN / "e8.npz")
    assert (rows, cols, tpg) == (8, 8, 12)
    assert np.array_equal(groups, e8["groups_12_2"])
    assert np.array_equal(tm, e8["tm_12_2"])
    assert vals.tobytes() == e8["values_12_2"].tobytes()
    assert np.array_equal(columns, e8["columns_12_2"])


@pytest.mark.parametrize("offset,byte,err", [(0, ord("X"), "FormatError"), (8, 0xEE, "FormatError"),
                                             (12, 9, "FormatError")])
def test_corrupted_header_rejected(argcsr, tmp_path, offset, byte, err):
    """test_io.cpp:163-182: bad magic, version or tag -> FormatError (before any device work)."""
    raw = bytearray((GOLDEN / "e8_argcsr_12_2.spfmt").read_bytes())
    raw[offset] = byte
    p = tmp_path / "bad.spfmt"
    p.write_bytes(bytes(raw))
    with pytest.raises(getattr(argcsr, err)):
        argcsr.read_binary(str(p))


@pytest.mark.parametrize("cut", [3, 12, 20, 60, 200, 452])
def test_truncated_stream_rejected(argcsr, tmp_path, cut):
    """test_io.cpp:184-190: truncation -> ParseError, also for a length prefix
    larger than the stream (no huge allocation)."""
    raw = (GOLDEN / "e8_argcsr_12_2.spfmt").read_bytes()
    p = tmp_path / "cut.spfmt"
    p.write_bytes(raw[:cut])
    with pytest.raises(argcsr.ParseError):
        argcsr.read_binary(str(p))


def test_unreadable_path(argcsr, tmp_path):
    with pytest.raises(argcsr.IoError):
        argcsr.read_binary(str(tmp_path / "missing.spfmt"))


def test_ellpack_container_unsupported(argcsr, tmp_path):
    p = tmp_path / "ell.spfmt"
    p.write_bytes(b"SPFMTBIN" + struct.pack("<IB", 1, 1) + struct.pack("<3Q", 1, 1, 1))
    with pytest.raises(argcsr.UnsupportedError):
        argcsr.read_binary(str(p))


# ---------------------------------------------------------------- on the GPU
@pytest.mark.gpu
@pytest.mark.parametrize("layout", LAYOUTS)
def test_write_binary_byte_identical(argcsr, tmp_path, layout):
    e8 = np.load(GOLDEN / "e8.npz")
    A = (8, 8, e8["e8_rp"], e8["e8_cols"], e8["e8_vals"])
    m = argcsr.argcsr_from_csr(A, 12, 2, layout=layout[0], x_remap=layout[1])
    argcsr.write_binary(str(tmp_path / "e8.spfmt"), m)
    assert (tmp_path / "e8.spfmt").read_bytes() == (GOLDEN / "e8_argcsr_12_2.spfmt").read_bytes()


@pytest.mark.gpu
@pytest.mark.parametrize("layout", LAYOUTS)
def test_write_binary_corpus_and_powerlaw_match_reference(argcsr, orc, ref, corpus, tmp_path, layout):
    cases = [(corpus[i], t, d) for i in (1, 3, 17, 42) for t, d in ((32, 4), (128, 1))]
    cases.append((powerlaw_csr(5000, 4000, seed=5, heavy_rows=[(3, 3000)]), 128, 1))
    for k, (A, t, d) in enumerate(cases):
        m = to_dev(argcsr, A, t, d, layout=layout)
        argcsr.write_binary(str(tmp_path / f"{k}.spfmt"), m)
        ref.write_binary(orc.argcsr_from_csr(A, t, d), str(tmp_path / f"{k}.ref"))
        assert (tmp_path / f"{k}.spfmt").read_bytes() == (tmp_path / f"{k}.ref").read_bytes(), (k, t, d)


@pytest.mark.gpu
@pytest.mark.parametrize("layout", LAYOUTS)
def test_read_binary_round_trip(argcsr, orc, tmp_path, layout):
    """The reference's container imported onto the device: same arrays, the
    SpMV bit-identical to the reference's spmv_argcsr on them."""
    for name in ("e8_argcsr_12_2.spfmt", "corpus3_argcsr_32_4.spfmt"):
        rows, cols, tpg, groups, tm, vals, columns = parse_argcsr_container((GOLDEN / name).read_bytes())
        m = argcsr.read_binary(str(GOLDEN / name), layout=layout[0], x_remap=layout[1])
        assert (m.num_rows, m.num_cols, m.threads_per_group) == (rows, cols, tpg)
        assert np.array_equal(m.groups_array, groups) and np.array_equal(m.threads_mapping, tm)
        assert np.array_equal(m.columns, columns) and m.values.tobytes() == vals.tobytes()
        x = np.linspace(-1, 2, cols)
        import oracle

        M = oracle.ArgCsr(rows, cols, tpg, groups.copy(), tm.copy(), vals.copy(), columns.copy())
        assert bits(argcsr.spmv(m, x)) == bits(orc.spmv_argcsr(M, x))
        argcsr.write_binary(str(tmp_path / name), m)
        assert (tmp_path / name).read_bytes() == (GOLDEN / name).read_bytes()


@pytest.mark.gpu
def test_read_binary_csr_container_converts(argcsr, orc):
    e8 = np.load(GOLDEN / "e8.npz")
    for t, d in ((12, 2), (12, 1), (4, 100)):
        m = argcsr.read_binary(str(GOLDEN / "e8_csr.spfmt"), threads_per_group=t, desired_chunk_size=d)
        assert np.array_equal(m.groups_array, e8[f"groups_{t}_{d}"])
        assert np.array_equal(m.columns, e8[f"columns_{t}_{d}"])


@pytest.mark.gpu
@pytest.mark.parametrize("layout", LAYOUTS)
def test_import_reference_arrays(argcsr, orc, layout):
    A = powerlaw_csr(8000, 6000, seed=21, heavy_rows=[(10, 4000)])
    for t, d in ((128, 1), (32, 4), (30, 3)):
        R = orc.argcsr_from_csr(A, t, d)
        m = argcsr.argcsr_from_reference(R.num_rows, R.num_cols, t, R.groups, R.threads_mapping, R.values,
                                         R.columns, layout=layout[0], x_remap=layout[1])
        assert_same_layout(m, R, f"import ({t},{d})")
        assert m.nnz == A.columns.size
        x = np.cos(np.arange(A.num_cols, dtype=np.float64))
        assert bits(argcsr.spmv(m, x)) == bits(orc.spmv_argcsr(R, x))


@pytest.mark.gpu
def test_import_rejects_broken_layouts(argcsr, orc):
    A = powerlaw_csr(500, 400, seed=2, max_len=60)
    R = orc.argcsr_from_csr(A, 32, 1)

    def attempt(groups=None, tm=None, values=None, columns=None, tpg=32):
        argcsr.argcsr_from_reference(R.num_rows, R.num_cols, tpg, R.groups if groups is None else groups,
                                     R.threads_mapping if tm is None else tm,
                                     R.values if values is None else values,
                                     R.columns if columns is None else columns)

    g = R.groups.copy()
    g[1, 2] += 32  # offset
    with pytest.raises(argcsr.FormatError):
        attempt(groups=g)
    tm = R.threads_mapping.copy()
    tm[0] = 0  # a row without a thread
    with pytest.raises(argcsr.FormatError):
        attempt(tm=tm)
    c = R.columns.copy()
    free = int(R.groups[0, 2] + R.threads_mapping[int(R.groups[0, 1]) - 1])  # first free lane of group 0, j = 0
    if free < int(R.groups[0, 2]) + 32:
        c[free] = 0  # an entry in a free lane
        with pytest.raises(argcsr.FormatError):
            attempt(columns=c)
    with pytest.raises(argcsr.FormatError):
        attempt(values=R.values[:-1], columns=R.columns[:-1])


# --------------------------------------------------------- Matrix Market (host)
MM_CASES = {
    "general": "%%MatrixMarket matrix coordinate real general\n% c\n3 4 5\n1 1 1.5\n3 4 -2\n2 2 0.25\n1 1 0.125\n3 1 1e-300\n",
    "symmetric": "%%MatrixMarket matrix coordinate real symmetric\n4 4 4\n1 1 2\n2 1 -1\n4 3 3.5\n3 2 0.1\n",
    "skew": "%%MatrixMarket matrix coordinate integer skew-symmetric\n3 3 2\n2 1 7\n3 1 -4\n",
    "pattern": "%%MatrixMarket matrix coordinate pattern general\n2 5 3\n1 5\n2 1\n1 2\n",
    "dups": "%%MatrixMarket matrix coordinate real general\n2 2 6\n1 1 0.1\n1 1 0.2\n1 1 0.3\n2 2 1\n2 2 -1\n1 2 -0.0\n",
}


@pytest.mark.parametrize("name", sorted(MM_CASES))
def test_matrix_market_matches_reference(argcsr, ref, tmp_path, name):
    """read_matrix_market (io.cpp:42-128) -- symmetric expansion, skew sign,
    pattern 1.0, 1-based indices, duplicate sums -- equals the reference's."""
    p = tmp_path / f"{name}.mtx"
    p.write_text(MM_CASES[name])
    A = argcsr.read_matrix_market(str(p))
    R = ref.read_matrix_market(str(p))
    assert (A.num_rows, A.num_cols) == (R.num_rows, R.num_cols)
    assert np.array_equal(A.row_pointers, R.row_pointers)
    assert np.array_equal(A.columns, R.columns)
    assert A.values.tobytes() == R.values.tobytes()


def test_matrix_market_round_trip_corpus(argcsr, ref, corpus, tmp_path):
    """write_matrix_market then read (ours and the reference's) reproduces the
    matrix exactly (17 significant digits, test_io.cpp:122-129)."""
    for i, R in enumerate(corpus[:25]):
        A = argcsr.CsrMatrix.from_arrays(R.num_rows, R.num_cols, R.row_pointers, R.columns, R.values)
        p = tmp_path / f"c{i}.mtx"
        argcsr.write_matrix_market(str(p), A)
        for B in (argcsr.read_matrix_market(str(p)), ref.read_matrix_market(str(p))):
            assert np.array_equal(B.row_pointers, R.row_pointers) and np.array_equal(B.columns, R.columns)
            assert B.values.tobytes() == R.values.tobytes()


@pytest.mark.parametrize("text,err", [
    ("", "ParseError"),
    ("%%MatrixMarket matrix array real general\n1 1\n1\n", "UnsupportedError"),
    ("%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1 0\n", "UnsupportedError"),
    ("%%MatrixMarket matrix coordinate real hermitian\n1 1 1\n1 1 1\n", "UnsupportedError"),
    ("%%MatrixMarket vector coordinate real general\n1 1 1\n1 1 1\n", "UnsupportedError"),
    ("%%NotMM matrix coordinate real general\n1 1 1\n1 1 1\n", "ParseError"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1\n", "ParseError"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1\n", "BoundsError"),
    ("%%MatrixMarket matrix coordinate real general\n0 2 0\n", "ParseError"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1\n", "ParseError"),
])
def test_matrix_market_errors(argcsr, tmp_path, text, err):
    p = tmp_path / "bad.mtx"
    p.write_text(text)
    with pytest.raises(getattr(argcsr, err)):
        argcsr.read_matrix_market(str(p))
    with pytest.raises(argcsr.IoError):
        argcsr.read_matrix_market(str(tmp_path / "missing.mtx"))


def test_csr_from_triplets_duplicate_order_matches_reference(argcsr, ref):
    """Many duplicates in a large unsorted entry list: the duplicate sums
    (whose rounding depends on the order the sort leaves equal keys in) are
    bit-identical to the reference csr_from_triplets (core.cpp:7-48)."""
    rng = np.random.default_rng(5)
    for n, k in ((7, 40), (30, 5000), (200, 20000)):
        ents = [(int(r), int(c), float(v)) for r, c, v in
                zip(rng.integers(0, n, k), rng.integers(0, n, k), rng.uniform(-1, 1, k) * 10.0 ** rng.integers(-8, 8, k))]
        A = argcsr.csr_from_triplets(n, n, ents)
        R = ref.csr_from_triplets(n, n, ents)
        assert np.array_equal(A.row_pointers, R.row_pointers) and np.array_equal(A.columns, R.columns)
        assert A.values.tobytes() == R.values.tobytes()
