"""CPU-only checks of the boundary: the C-ABI library loads and exports every
symbol include/argcsr_gpu.h declares, the pybind module mirrors the reference
module's API, argument validation follows the reference's order (no device
needed for those), and a missing device fails loudly (no CPU fallback)."""
import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent


def declared_symbols():
    text = (ROOT / "include" / "argcsr_gpu.h").read_text()
    return sorted(set(re.findall(r"ARGCSR_API\s+[\w\s\*]+?\b(argcsr_\w+)\s*\(", text)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ("argcsr_dev_convert", "argcsr_dev_export", "argcsr_dev_spmv", "argcsr_dev_spmv_groups",
              "argcsr_dev_spmv_host", "argcsr_dev_to_csr", "argcsr_dev_chunk_entries", "argcsr_dev_padding_stats",
              "argcsr_dev_free", "argcsr_last_error", "argcsr_partition_rows"):
        assert s in syms


def test_c_abi_library_exports_every_declared_symbol(argcsr):
    lib = ctypes.CDLL(argcsr.native_library_path())
    for s in declared_symbols():
        assert hasattr(lib, s), f"{s} not exported"
    lib.argcsr_abi_version.restype = ctypes.c_int
    assert lib.argcsr_abi_version() == 2


def test_library_is_sm100a():
    import subprocess

    lib = ROOT / "paper_1203_5737_b200" / "libargcsr_gpu.so"
    out = subprocess.run(["cuobjdump", "--list-elf", str(lib)], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_c_abi_parameter_errors_without_device():
    lib = ctypes.CDLL(str(ROOT / "paper_1203_5737_b200" / "libargcsr_gpu.so"))

    class View(ctypes.Structure):
        _fields_ = [("num_rows", ctypes.c_uint64), ("num_cols", ctypes.c_uint64), ("nnz", ctypes.c_uint64),
                    ("row_pointers", ctypes.c_void_p), ("columns", ctypes.c_void_p), ("values", ctypes.c_void_p),
                    ("dtype", ctypes.c_int), ("space", ctypes.c_int)]

    lib.argcsr_last_error.restype = ctypes.c_char_p
    rp = np.array([0, 1], np.uint64)
    cols = np.array([0], np.int32)
    vals = np.array([1.0])
    v = View(1, 1, 1, rp.ctypes.data, cols.ctypes.data, vals.ctypes.data, 0, 0)
    out = ctypes.c_void_p()
    # argcsr.cpp:20-23: parameters checked first
    assert lib.argcsr_dev_convert(ctypes.byref(v), 0, 1, 0, None, ctypes.byref(out)) == 1
    assert b"threads_per_group and desired_chunk_size" in lib.argcsr_last_error()
    assert lib.argcsr_dev_convert(ctypes.byref(v), 4, 0, 0, None, ctypes.byref(out)) == 1
    # argcsr.cpp:24-26: empty row set
    v.num_rows = 0
    assert lib.argcsr_dev_convert(ctypes.byref(v), 4, 1, 0, None, ctypes.byref(out)) == 1
    assert b"row_nnz must be nonempty" in lib.argcsr_last_error()
    # device limit
    v.num_rows = 1
    assert lib.argcsr_dev_convert(ctypes.byref(v), 16385, 1, 0, None, ctypes.byref(out)) == 11


def test_module_api_mirrors_reference(argcsr):
    for name in ("CsrMatrix", "GroupInfo", "ArgCsrMatrix", "FormatStats", "Error", "csr_from_triplets",
                 "triplets_from_csr", "argcsr_from_csr", "csr_from_argcsr", "spmv", "padding_stats",
                 "chunk_entries"):
        assert hasattr(argcsr, name)
    assert argcsr.kDefaultThreadsPerGroup == 128 and argcsr.kDefaultDesiredChunkSize == 1
    for cls in (argcsr.ParameterError, argcsr.DimensionError, argcsr.BoundsError, argcsr.CudaError):
        assert issubclass(cls, argcsr.Error)


def test_triplets_round_trip(argcsr):  # python/test_smoke.py:15-18
    a = argcsr.csr_from_triplets(3, 3, [(2, 0, -1.0), (0, 1, 2.0), (0, 1, 3.0)])
    assert a.nnz == 2
    assert argcsr.triplets_from_csr(a) == [(0, 1, 5.0), (2, 0, -1.0)]


def test_csr_from_triplets_matches_reference(argcsr, ref):
    rng = np.random.default_rng(3)
    for _ in range(20):
        nr, nc = int(rng.integers(1, 40)), int(rng.integers(1, 40))
        n = int(rng.integers(0, 200))
        ent = [(int(rng.integers(0, nr)), int(rng.integers(0, nc)), float(rng.uniform(-1, 1))) for _ in range(n)]
        mine = argcsr.csr_from_triplets(nr, nc, ent)
        want = ref.csr_from_triplets(nr, nc, ent)
        assert np.array_equal(mine.row_pointers, want.row_pointers)
        assert np.array_equal(mine.columns, want.columns)
        assert mine.values.tobytes() == want.values.tobytes()


def test_errors_surface_as_exceptions_without_device(argcsr):  # python/test_smoke.py:64-70
    with pytest.raises(argcsr.Error):
        argcsr.csr_from_triplets(2, 2, [(5, 0, 1.0)])
    a = argcsr.csr_from_triplets(2, 2, [(0, 0, 1.0)])
    with pytest.raises(argcsr.ParameterError):
        argcsr.argcsr_from_csr(a, threads_per_group=0)
    with pytest.raises(argcsr.UnsupportedError):
        argcsr.spmv(a, [1.0, 2.0])  # CSR SpMV is not on the device path


def test_no_cpu_fallback(argcsr):
    import torch

    if torch.cuda.is_available():
        pytest.skip("device present")
    a = argcsr.csr_from_triplets(2, 2, [(0, 0, 1.0)])
    with pytest.raises(argcsr.CudaError):
        argcsr.argcsr_from_csr(a, 4, 1)


def test_partition_rows_nnz_balanced(argcsr):
    rp = np.array([0, 10, 10, 10, 30, 31, 60, 61, 62, 100], np.uint64)
    for parts in (1, 2, 3, 4, 9):
        b = argcsr.partition_rows(rp, parts)
        assert b[0] == 0 and b[-1] == 9 and np.all(np.diff(b.astype(np.int64)) >= 1)
    b = argcsr.partition_rows(rp, 2)
    assert b[1] == np.searchsorted(rp, 50)


def _build_example(tmp_path):
    import subprocess

    root = Path(__file__).resolve().parent.parent
    exe = tmp_path / "spmv_example"
    cmd = ["g++", "-std=c++20", "-O2", f"-I{root / 'include'}", str(root / "examples" / "spmv_example.cpp"),
           f"-L{root / 'paper_1203_5737_b200'}", "-largcsr_gpu", f"-Wl,-rpath,{root / 'paper_1203_5737_b200'}",
           "-o", str(exe)]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return exe


def test_cpp_example_builds_and_fails_loudly_without_a_device(tmp_path):
    """include/argcsr_gpu.hpp is a usable C++ API over the C-ABI library; with
    no CUDA device the product path raises (no CPU fallback)."""
    import subprocess

    import torch

    exe = _build_example(tmp_path)
    if torch.cuda.is_available():
        pytest.skip("a device is present (tests/test_gpu_parity.py runs the example)")
    r = subprocess.run([str(exe), "16"], capture_output=True, text=True)
    assert r.returncode == 2 and "no CUDA device" in r.stderr


@pytest.mark.gpu
def test_cpp_example_runs_on_the_device(tmp_path):
    import subprocess

    exe = _build_example(tmp_path)
    r = subprocess.run([str(exe), "300", str(tmp_path / "a.spfmt")], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "lossless=1" in r.stdout


def test_peer_needed_rows_are_the_halo():
    """The rows each rank reads from every other slice (argcsr_plan_needed,
    the halo plan of the multi-GPU layer): for a 27-pt stencil split 4 ways,
    about one plane of each neighbour, nothing from the others."""
    from helpers import stencil27
    from paper_1203_5737_b200.multigpu import needed_rows, partition_bounds

    n = 16
    A = stencil27(n)
    b = partition_bounds(A.row_pointers, 4)
    for p in range(4):
        a0, a1 = int(A.row_pointers[b[p]]), int(A.row_pointers[b[p + 1]])
        cols = np.asarray(A.columns[a0:a1])
        need = needed_rows(cols, A.num_cols, b, p)
        assert len(need[p]) == 0
        for q in range(4):
            if abs(q - p) > 1:
                assert len(need[q]) == 0
            elif q != p:
                assert 0 < len(need[q]) <= n * n + n + 1  # one plane (+ one row and one point of the next)
                inq = np.unique(cols[(cols >= b[q]) & (cols < b[q + 1])])
                assert np.array_equal(need[q], inq.astype(np.uint64))


def test_peer_abi_parameter_errors_without_device(argcsr):
    import paper_1203_5737_b200._argcsr_gpu as ext

    with pytest.raises(argcsr.ParameterError):
        ext.peer_signal([1] * 8, 1)  # at most 7 peers
    with pytest.raises(argcsr.ParameterError):
        ext.peer_signal([1, 2], 1, 0, [3])  # one partial destination per flag
    with pytest.raises(argcsr.ParameterError):
        ext.peer_open(b"short", 0)
