"""The CPU oracle (oracle/argcsr_oracle.c) pinned against the reference:
golden fixtures generated from the compiled reference (tests/golden/), the
literal known-answer tests of proj/tests/test_argcsr.cpp, and — when
oracle/_ref is built — the compiled reference itself over the whole
500-matrix corpus x (tpg, dcs) grid."""
import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

import oracle
from oracle import Csr

GOLD = Path(__file__).resolve().parent / "golden"


def digest_case(M, y) -> str:
    h = hashlib.sha256()
    for a in (M.groups.astype("<u8"), M.threads_mapping.astype("<u8"), M.values.astype("<f8"),
              M.columns.astype("<i4"), np.asarray(y, "<f8")):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def corpus_digest(orc, A, grid, x):
    h = hashlib.sha256()
    for t, d in grid:
        M = orc.argcsr_from_csr(A, t, d)
        h.update(digest_case(M, orc.spmv_argcsr(M, x)).encode())
    return h.hexdigest()[:32]


def probe_vector(n, salt=0):  # proj/tests/support.hpp:74-81
    j = np.arange(n, dtype=np.int64)
    return 1.0 + 0.0625 * ((j + salt) % 17).astype(np.float64) - 0.25 * (j % 3).astype(np.float64)


# ------------------------------------------------------------ known answers
def test_partition_known_answers(orc):  # test_argcsr.cpp:9-36
    assert orc.partition_groups([1, 1, 1, 1, 1, 1, 1, 8], 12, 1).tolist() == [[0, 7], [7, 1]]
    assert orc.partition_groups([5, 5, 5], 2, 100).tolist() == [[0, 2], [2, 1]]
    assert orc.partition_groups([1000], 4, 1).tolist() == [[0, 1]]
    assert orc.partition_groups([1000, 1], 4, 1).tolist() == [[0, 1], [1, 1]]
    assert orc.partition_groups([1, 1000, 1], 4, 1).tolist() == [[0, 1], [1, 1], [2, 1]]
    for bad in (([1], 0, 1), ([1], 4, 0), ([], 4, 1)):
        with pytest.raises(oracle.OracleError):
            orc.partition_groups(*bad)


def test_assign_threads_known_answers(orc):  # test_argcsr.cpp:38-89
    tpr, ch, asg, fr = orc.assign_threads([1, 1, 1, 1, 1, 1, 1, 8], 12)
    assert tpr.tolist() == [1, 1, 1, 1, 1, 1, 1, 4] and (ch, asg, fr) == (2, 11, 1)
    tpr, ch, _, fr = orc.assign_threads([5], 4)
    assert tpr.tolist() == [3] and (ch, fr) == (2, 1)
    tpr, ch, _, fr = orc.assign_threads([2, 2, 2, 2], 4)
    assert tpr.tolist() == [1, 1, 1, 1] and (ch, fr) == (2, 0)
    tpr, ch, _, fr = orc.assign_threads([1000], 4)
    assert tpr.tolist() == [4] and (ch, fr) == (250, 0)
    tpr, ch, _, _ = orc.assign_threads([0], 4)
    assert tpr.tolist() == [1] and ch == 0
    tpr, ch, _, fr = orc.assign_threads([0, 3], 4)
    assert tpr.tolist() == [1, 3] and (ch, fr) == (1, 0)
    with pytest.raises(oracle.OracleError):
        orc.assign_threads([1, 1, 1], 2)


def test_spmv_validates_length(orc):
    g = np.load(GOLD / "e8.npz")
    A = Csr(8, 8, g["e8_rp"], g["e8_cols"], g["e8_vals"])
    M = orc.argcsr_from_csr(A, 12, 2)
    with pytest.raises(oracle.OracleError):
        orc.spmv_argcsr(M, np.ones(7))


# ------------------------------------------------------------ golden fixtures
def test_e8_golden(orc):
    g = np.load(GOLD / "e8.npz")
    A = Csr(8, 8, g["e8_rp"], g["e8_cols"], g["e8_vals"])
    x = 1.0 + 0.25 * np.arange(8)
    for key in [k[len("groups_"):] for k in g.files if k.startswith("groups_")]:
        t, d = map(int, key.split("_"))
        M = orc.argcsr_from_csr(A, t, d)
        assert np.array_equal(M.groups, g[f"groups_{key}"]), key
        assert np.array_equal(M.threads_mapping, g[f"tm_{key}"]), key
        assert M.values.tobytes() == g[f"values_{key}"].tobytes(), key
        assert np.array_equal(M.columns, g[f"columns_{key}"]), key
        assert orc.spmv_argcsr(M, x).tobytes() == g[f"y_{key}"].tobytes(), key
    # the anatomy the reference tests spell out (test_argcsr.cpp:91-121)
    assert g["groups_12_2"].tolist() == [[0, 8, 0, 2]]
    assert g["tm_12_2"].tolist() == [1, 2, 3, 4, 5, 6, 7, 11]
    assert g["groups_12_1"].tolist() == [[0, 7, 0, 1], [7, 1, 12, 2]]
    assert g["tm_12_1"].tolist() == [1, 2, 3, 4, 5, 6, 7, 4]


def test_corpus40_golden(orc):
    g = np.load(GOLD / "corpus40.npz")
    digests = json.loads((GOLD / "corpus_digests.json").read_text())
    grid = [tuple(p) for p in digests["grid"]]
    for i in range(40):
        nr, nc = (int(v) for v in g[f"{i}_shape"])
        A = Csr(nr, nc, g[f"{i}_rp"], g[f"{i}_cols"], g[f"{i}_vals"])
        x = probe_vector(nc)
        if i < 10:
            for t, d in ((4, 1), (32, 4), (128, 1), (12, 2)):
                k = f"{i}_{t}_{d}"
                M = orc.argcsr_from_csr(A, t, d)
                assert np.array_equal(M.groups, g[f"{k}_groups"]) and np.array_equal(M.columns, g[f"{k}_columns"])
                assert M.values.tobytes() == g[f"{k}_values"].tobytes()
                assert np.array_equal(M.threads_mapping, g[f"{k}_tm"])
                assert orc.spmv_argcsr(M, x).tobytes() == g[f"{k}_y"].tobytes()
        assert corpus_digest(orc, A, grid, x) == digests["digests"][str(i)], f"corpus[{i}]"


def test_full_corpus_digests_against_compiled_reference(orc, ref, corpus):
    """All 500 corpus matrices (generated by the compiled reference) x the
    full grid: oracle == golden digests == compiled reference."""
    digests = json.loads((GOLD / "corpus_digests.json").read_text())
    grid = [tuple(p) for p in digests["grid"]]
    g = np.load(GOLD / "corpus40.npz")
    for i in range(40):  # the stored inputs are the reference corpus
        assert np.array_equal(corpus[i].row_pointers, g[f"{i}_rp"])
        assert corpus[i].values.tobytes() == g[f"{i}_vals"].tobytes()
    for i, A in enumerate(corpus):
        x = ref.probe_vector(A.num_cols)
        assert np.array_equal(x, probe_vector(A.num_cols))
        assert corpus_digest(orc, A, grid, x) == digests["digests"][str(i)], f"corpus[{i}]"


def test_oracle_pieces_match_reference(orc, ref):
    rng = np.random.default_rng(11)
    for _ in range(300):
        n = int(rng.integers(1, 60))
        counts = rng.integers(0, 400, n)
        counts[rng.random(n) < 0.2] = 0
        t = int(rng.integers(1, 160))
        d = int(rng.integers(1, 40))
        assert np.array_equal(orc.partition_groups(counts, t, d), ref.partition_groups(counts, t, d))
        if n <= t:
            a, b = orc.assign_threads(counts, t), ref.assign_threads(counts, t)
            assert np.array_equal(a[0], b[0]) and a[1:] == b[1:]


def test_parallel_spmv_is_bit_identical(orc, corpus):  # test_bench.cpp:43-71, acceptance criterion 5
    for A in corpus[:50]:
        M = orc.argcsr_from_csr(A)
        x = probe_vector(A.num_cols)
        assert orc.spmv_argcsr_parallel(M, x, 5).tobytes() == orc.spmv_argcsr(M, x).tobytes()


def test_round_trip_and_bound(orc, corpus):  # acceptance criteria 3-4
    for A in corpus[:100]:
        x = probe_vector(A.num_cols)
        y_csr = orc.spmv_csr(A, x)
        absrow = orc.abs_row_sums(A, x)
        for t, d in ((4, 1), (32, 4), (128, 32)):
            M = orc.argcsr_from_csr(A, t, d)
            B = orc.csr_from_argcsr(M)
            assert np.array_equal(B.row_pointers, A.row_pointers) and np.array_equal(B.columns, A.columns)
            assert np.all(np.abs(orc.spmv_argcsr(M, x) - y_csr) <= 1e-12 * absrow)
