"""B200-native ARG-CSR (Adaptive Row-grouped CSR, arXiv 1203.5737).

Drop-in for the hot path of the reference `argcsr` Python module
(proj/python/bindings.cpp): CSR -> ARG-CSR conversion and ARG-CSR SpMV run as
hand-written sm_100a kernels behind the C-ABI in include/argcsr_gpu.h.  The
names, argument names, defaults and error classes follow the reference:

    >>> import paper_1203_5737_b200 as argcsr
    >>> a = argcsr.csr_from_triplets(8, 8, entries)
    >>> m = argcsr.argcsr_from_csr(a, threads_per_group=12, desired_chunk_size=2)
    >>> m.groups, m.threads_mapping, m.values, m.columns   # reference layout, bit-exact
    >>> y = argcsr.spmv(m, x)                              # bit-identical to spmv_argcsr

The converted matrix lives in device memory; its reference-layout arrays are
exported lazily.  There is no CPU fallback: without the native extension or a
CUDA device every compute call raises.
"""
from __future__ import annotations

import numpy as _np

from ._errors import (  # noqa: F401
    BoundsError,
    CorrectnessError,
    CudaError,
    DimensionError,
    Error,
    FormatError,
    InternalError,
    IoError,
    NcclError,
    OutOfMemoryError,
    ParameterError,
    ParseError,
    UnsupportedError,
)

try:
    from . import _argcsr_gpu as _ext
except ImportError as exc:  # fail loudly: the product path is native only
    raise ImportError(
        "paper_1203_5737_b200: native extension missing; build it with "
        "`python paper_1203_5737_b200/_build.py` (or __graft_entry__.build())"
    ) from exc

CsrMatrix = _ext.CsrMatrix
GroupInfo = _ext.GroupInfo
FormatStats = _ext.FormatStats
ArgCsrMatrix = _ext.ArgCsrMatrix
EllpackMatrix = _ext.EllpackMatrix
SlicedEllpackMatrix = _ext.SlicedEllpackMatrix
ellpack_from_csr = _ext.ellpack_from_csr
sliced_from_csr = _ext.sliced_from_csr
csr_from_ellpack = _ext.csr_from_ellpack
csr_from_sliced = _ext.csr_from_sliced

kDefaultThreadsPerGroup = _ext.kDefaultThreadsPerGroup
kDefaultDesiredChunkSize = _ext.kDefaultDesiredChunkSize
kPaddingColumn = _ext.kPaddingColumn

csr_from_triplets = _ext.csr_from_triplets
triplets_from_csr = _ext.triplets_from_csr
csr_from_argcsr = _ext.csr_from_argcsr
csr_arrays_from_argcsr = _ext.csr_arrays_from_argcsr
chunk_entries = _ext.chunk_entries
padding_stats = _ext.padding_stats
balance_stats = _ext.balance_stats
BalanceStats = _ext.BalanceStats
read_matrix_market = _ext.read_matrix_market
write_matrix_market = _ext.write_matrix_market
partition_rows = _ext.partition_rows
abi_version = _ext.abi_version


# argcsr_dev_convert_ex flags (include/argcsr_gpu.h)
LAYOUTS = {"compact": 0, "reference": 1}
X_REMAP = {"auto": 0, "on": 2, "off": 4}


def _layout_flags(layout: str, x_remap: str = "auto") -> int:
    if layout not in LAYOUTS:
        raise ParameterError(f"argcsr_from_csr: layout must be one of {sorted(LAYOUTS)}")
    if x_remap not in X_REMAP:
        raise ParameterError(f"argcsr_from_csr: x_remap must be one of {sorted(X_REMAP)}")
    return LAYOUTS[layout] | X_REMAP[x_remap]


def argcsr_from_csr(matrix, threads_per_group: int = kDefaultThreadsPerGroup,
                    desired_chunk_size: int = kDefaultDesiredChunkSize, device: int = 0,
                    layout: str = "compact", x_remap: str = "auto") -> ArgCsrMatrix:
    """argcsr_from_csr (argcsr.hpp:101-104) on the GPU.

    `matrix` is a CsrMatrix, or a tuple (num_rows, num_cols, row_pointers,
    columns, values) of numpy arrays (float32 values give an fp32 handle), or
    a dict of torch CUDA tensors (see argcsr_from_torch).  `layout` picks the
    device storage of the value/column blocks: "compact" (free lanes not
    stored, the default) or "reference" (the reference arrays verbatim); the
    exported arrays and every SpMV result are identical either way.
    `x_remap` ("auto" | "on" | "off") controls the device-internal column
    order that keeps x's working set L2-resident (compact layout only).
    """
    flags = _layout_flags(layout, x_remap)
    if isinstance(matrix, CsrMatrix):
        return _ext.argcsr_from_csr(matrix, threads_per_group, desired_chunk_size, device, flags)
    if isinstance(matrix, tuple) and len(matrix) == 5:
        nr, nc, rp, cols, vals = matrix
        return _ext.argcsr_from_csr_arrays(nr, nc, rp, cols, vals, threads_per_group, desired_chunk_size, device,
                                           flags)
    raise ParameterError("argcsr_from_csr: expected a CsrMatrix or (num_rows, num_cols, rp, cols, vals)")


def argcsr_from_torch(num_rows: int, num_cols: int, row_pointers, columns, values,
                      threads_per_group: int = kDefaultThreadsPerGroup,
                      desired_chunk_size: int = kDefaultDesiredChunkSize, stream=None,
                      layout: str = "compact", x_remap: str = "auto") -> ArgCsrMatrix:
    """Convert a device-resident CSR given as torch CUDA tensors (int64 row
    pointers, int32 columns, float64/float32 values) on the current stream."""
    import torch

    flags = _layout_flags(layout, x_remap)
    if not (row_pointers.is_cuda and columns.is_cuda and values.is_cuda):
        raise ParameterError("argcsr_from_torch: tensors must be CUDA tensors")
    if row_pointers.dtype != torch.int64 or columns.dtype != torch.int32:
        raise ParameterError("argcsr_from_torch: row_pointers int64 and columns int32 required")
    if values.dtype not in (torch.float64, torch.float32):
        raise ParameterError("argcsr_from_torch: values must be float64 or float32")
    if row_pointers.numel() != num_rows + 1 or columns.numel() != values.numel():
        raise DimensionError("argcsr_from_torch: array lengths do not match")
    dev = values.device.index
    s = stream if stream is not None else torch.cuda.current_stream(values.device)
    dtype = "float64" if values.dtype == torch.float64 else "float32"
    return _ext.argcsr_from_device_csr(
        num_rows, num_cols, values.numel(), row_pointers.contiguous().data_ptr(), columns.contiguous().data_ptr(),
        values.contiguous().data_ptr(), dtype, threads_per_group, desired_chunk_size, dev, s.cuda_stream, flags)


def write_binary(path: str, matrix: ArgCsrMatrix) -> None:
    """write_binary(path, matrix) (bindings.cpp:168-171 -> io.cpp:282-298):
    the reference's SPFMTBIN container, byte-identical to the reference's."""
    _ext.write_binary(str(path), matrix)


def read_binary(path: str, threads_per_group: int = kDefaultThreadsPerGroup,
                desired_chunk_size: int = kDefaultDesiredChunkSize, device: int = 0, layout: str = "compact",
                x_remap: str = "auto") -> ArgCsrMatrix:
    """read_binary(path) (bindings.cpp:172 -> io.cpp:300-366) onto the device:
    an ARG-CSR container is imported as stored (a cached conversion); a CSR
    container is converted with threads_per_group / desired_chunk_size."""
    return _ext.read_binary(str(path), threads_per_group, desired_chunk_size, device, _layout_flags(layout, x_remap))


def argcsr_from_reference(num_rows: int, num_cols: int, threads_per_group: int, groups, threads_mapping, values,
                          columns, device: int = 0, layout: str = "compact", x_remap: str = "auto") -> ArgCsrMatrix:
    """A device handle from the reference ArgCsrMatrix arrays (groups as a
    G x 4 array of first_row, size, offset, chunk_size), checked, without
    re-running the converter."""
    return _ext.argcsr_from_reference_arrays(num_rows, num_cols, threads_per_group, groups, threads_mapping, values,
                                             columns, device, _layout_flags(layout, x_remap))


def spmv(matrix: ArgCsrMatrix, x):
    """spmv(matrix, x) (bindings.cpp:135 -> spmv_argcsr, argcsr.cpp:219-227).

    A list gives a list (the reference's behaviour), a numpy array gives a
    numpy array, a torch CUDA tensor gives a torch CUDA tensor (stream-ordered
    on the current stream).  A wrong length raises DimensionError.
    """
    if isinstance(matrix, (EllpackMatrix, SlicedEllpackMatrix)):  # ellpack.cpp:132-176
        host = _ext.spmv_ellpack_host if isinstance(matrix, EllpackMatrix) else _ext.spmv_sliced_host
        if type(x).__module__.startswith("torch"):
            return spmv_torch(matrix, x)
        if isinstance(x, _np.ndarray):
            return host(matrix, x)
        return host(matrix, _np.asarray(x, dtype=_np.float64)).tolist()
    if not isinstance(matrix, ArgCsrMatrix):
        raise UnsupportedError("spmv: only the device formats (ARG-CSR, ELLPACK, sliced ELLPACK) run here; "
                               "convert with argcsr_from_csr")
    mod = type(x).__module__
    if mod.startswith("torch"):
        return spmv_torch(matrix, x)
    if isinstance(x, _np.ndarray):
        return _ext.spmv_host(matrix, x)
    return _ext.spmv_host(matrix, _np.asarray(x, dtype=_np.float64)).tolist()


def spmv_torch(matrix: ArgCsrMatrix, x, out=None, stream=None):
    """y = A x for torch CUDA tensors, launched on `stream` (default: current)."""
    import torch

    want = torch.float64 if getattr(matrix, "dtype", "float64") == "float64" else torch.float32
    if not x.is_cuda or x.dtype != want:
        raise ParameterError(f"spmv: x must be a CUDA {want} tensor")
    if x.numel() != matrix.num_cols:
        raise DimensionError(f"spmv_argcsr: vector length {x.numel()} does not match {matrix.num_cols} columns")
    x = x.contiguous()
    y = out if out is not None else torch.empty(matrix.num_rows, dtype=want, device=x.device)
    if y.numel() != matrix.num_rows or y.dtype != want or not y.is_contiguous():
        raise DimensionError("spmv: output must be a contiguous vector of num_rows entries")
    s = stream if stream is not None else torch.cuda.current_stream(x.device)
    matrix.spmv_device(x.data_ptr(), y.data_ptr(), s.cuda_stream)
    return y


def spmv_argcsr_groups(matrix: ArgCsrMatrix, x, group_begin: int, group_end: int, y, stream=None):
    """spmv_argcsr_groups (argcsr.hpp:114-116) on torch CUDA tensors: writes
    only the rows of groups [group_begin, group_end) into y."""
    import torch

    s = stream if stream is not None else torch.cuda.current_stream(x.device)
    matrix.spmv_groups_device(x.data_ptr(), group_begin, group_end, y.data_ptr(), s.cuda_stream)
    return y


def native_library_path() -> str:
    """Path of the C-ABI shared library backing this module."""
    from pathlib import Path

    return str(Path(__file__).resolve().parent / "libargcsr_gpu.so")
