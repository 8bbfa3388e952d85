#!/usr/bin/env python
"""Generate the golden fixtures from the COMPILED REFERENCE (oracle/_ref,
built from /root/reference/proj/src/*.cpp by oracle/Makefile).

  python tests/golden/make_golden.py

Writes, next to this script:
  e8.npz               the E8 fixture (proj/tests/support.hpp:46-51) converted at
                       the (tpg, dcs) pairs the reference tests use, full arrays,
                       plus spmv_argcsr with x = 1 + 0.25 j
  corpus40.npz         CSR inputs of corpus[0:40] (support.hpp:86-119; libstdc++
                       RNG, so they are stored, not regenerated) and, for the
                       first 10 and (tpg, dcs) in SMALL_GRID, the full
                       conversion arrays and spmv_argcsr(probe_vector)
  corpus_digests.json  for all 500 corpus matrices, a digest of the reference
                       conversion + SpMV over the full GRID (checksum of checksums)
  *.spfmt              the reference's binary container (io.cpp:242-298) as
                       written by write_binary_file: e8 at (12, 2) and corpus[3]
                       at (32, 4) as ARG-CSR, e8 as CSR
"""
import hashlib
import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))

GRID = [(t, d) for t in (1, 3, 4, 12, 32, 128) for d in (1, 2, 4, 32)]
SMALL_GRID = [(4, 1), (32, 4), (128, 1), (12, 2)]
E8_PARAMS = [(12, 2), (12, 1), (14, 1), (15, 1), (128, 1), (8, 8), (4, 100)]


def digest_case(M, y) -> str:
    h = hashlib.sha256()
    for a in (M.groups.astype("<u8"), M.threads_mapping.astype("<u8"), M.values.astype("<f8"),
              M.columns.astype("<i4"), np.asarray(y, "<f8")):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def main():
    import oracle

    ref = oracle.ref()
    out = {}
    A = ref.e8()
    x8 = 1.0 + 0.25 * np.arange(8)
    out["e8_rp"], out["e8_cols"], out["e8_vals"] = A.row_pointers, A.columns, A.values
    for t, d in E8_PARAMS:
        M = ref.argcsr_from_csr(A, t, d)
        k = f"{t}_{d}"
        out[f"groups_{k}"], out[f"tm_{k}"] = M.groups, M.threads_mapping
        out[f"values_{k}"], out[f"columns_{k}"] = M.values, M.columns
        out[f"y_{k}"] = ref.spmv_argcsr(M, x8)
    np.savez_compressed(HERE / "e8.npz", **out)
    ref.write_binary(ref.argcsr_from_csr(A, 12, 2), str(HERE / "e8_argcsr_12_2.spfmt"))
    ref.write_binary_csr(A, str(HERE / "e8_csr.spfmt"))

    corpus = ref.corpus(500)
    ref.write_binary(ref.argcsr_from_csr(corpus[3], 32, 4), str(HERE / "corpus3_argcsr_32_4.spfmt"))
    c40 = {}
    for i, A in enumerate(corpus[:40]):
        c40[f"{i}_shape"] = np.array([A.num_rows, A.num_cols], np.uint64)
        c40[f"{i}_rp"], c40[f"{i}_cols"], c40[f"{i}_vals"] = A.row_pointers, A.columns, A.values
        if i >= 10:
            continue  # inputs only; corpus_digests.json pins their outputs
        x = ref.probe_vector(A.num_cols)
        for t, d in SMALL_GRID:
            M = ref.argcsr_from_csr(A, t, d)
            k = f"{i}_{t}_{d}"
            c40[f"{k}_groups"], c40[f"{k}_tm"] = M.groups, M.threads_mapping
            c40[f"{k}_values"], c40[f"{k}_columns"] = M.values, M.columns
            c40[f"{k}_y"] = ref.spmv_argcsr(M, x)
    np.savez_compressed(HERE / "corpus40.npz", **c40)

    digests = {}
    for i, A in enumerate(corpus):
        h = hashlib.sha256()
        x = ref.probe_vector(A.num_cols)
        for t, d in GRID:
            M = ref.argcsr_from_csr(A, t, d)
            h.update(digest_case(M, ref.spmv_argcsr(M, x)).encode())
        digests[str(i)] = h.hexdigest()[:32]
    (HERE / "corpus_digests.json").write_text(json.dumps(
        {"grid": GRID, "seed": 20260822, "count": 500, "digests": digests}, indent=0))


if __name__ == "__main__":
    main()
