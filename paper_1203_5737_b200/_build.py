"""In-tree build of the native pieces (no JIT cache: the .so files travel with
the repo snapshot to the GPU box).

  libargcsr_gpu.so        nvcc, sm_100a: CUDA kernels + the C-ABI (include/argcsr_gpu.h)
  _argcsr_gpu.<abi>.so    g++, pybind11 module over the C-ABI (rpath $ORIGIN)

Rebuilds only when a source is newer than its output.
"""
from __future__ import annotations

import os
import subprocess
import sysconfig
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
INCLUDE = ROOT / "include"

CUDA_SOURCES = ["capi.cu", "convert.cu", "spmv.cu", "inverse.cu", "xremap.cu", "ellpack.cu", "mgpu.cu"]
CUDA_HEADERS = ["common.cuh", "scan.cuh", "convert.cuh", "spmv.cuh", "inverse.cuh", "xremap.cuh", "ellpack.cuh"]
LIB = PKG / "libargcsr_gpu.so"
EXT = PKG / ("_argcsr_gpu" + (sysconfig.get_config_var("EXT_SUFFIX") or ".so"))

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo", "-O3", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
    "-Xptxas", "-v",
]


def _nccl_include() -> str:
    """nccl.h for the multi-GPU layer (types only: libnccl is dlopen'ed at run time)."""
    try:
        import nvidia.nccl

        p = Path(list(nvidia.nccl.__path__)[0]) / "include"
        if (p / "nccl.h").exists():
            return str(p)
    except Exception:
        pass
    return "/usr/include"


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or Path(cand).exists()):
            return cand
    return "nvcc"


def _stale(out: Path, deps: list[Path]) -> bool:
    if not out.exists():
        return True
    t = out.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def _run(cmd: list[str], log: Path | None = None) -> None:
    res = subprocess.run(cmd, capture_output=True, text=True)
    if log is not None:
        log.write_text(res.stdout + res.stderr)
    if res.returncode != 0:
        raise RuntimeError(f"build failed: {' '.join(cmd)}\n{res.stdout}\n{res.stderr}")


def build_lib(force: bool = False) -> Path:
    deps = [CSRC / s for s in CUDA_SOURCES + CUDA_HEADERS] + [INCLUDE / "argcsr_gpu.h"]
    if force or _stale(LIB, deps):
        # Export only the C-ABI: -fvisibility=hidden hides internals, the
        # header marks nothing, so re-export the argcsr_* symbols explicitly.
        cmd = [_nvcc(), *NVCC_FLAGS, "-shared", f"-I{INCLUDE}", f"-I{_nccl_include()}", "-o", str(LIB),
               *[str(CSRC / s) for s in CUDA_SOURCES],
               "-Xlinker", f"--version-script={CSRC / 'exports.map'}", "-ldl"]
        _run(cmd, PKG / "build_ptxas.log")
    return LIB


def build_ext(force: bool = False) -> Path:
    import pybind11

    deps = [CSRC / "bindings.cpp", CSRC / "host_io.hpp", INCLUDE / "argcsr_gpu.hpp", INCLUDE / "argcsr_gpu.h", LIB]
    if force or _stale(EXT, deps):
        py_inc = sysconfig.get_paths()["include"]
        cmd = ["g++", "-O2", "-std=c++20", "-shared", "-fPIC", "-fvisibility=hidden",
               f"-I{INCLUDE}", f"-I{pybind11.get_include()}", f"-I{py_inc}",
               str(CSRC / "bindings.cpp"), "-o", str(EXT),
               f"-L{PKG}", "-largcsr_gpu", "-Wl,-rpath,$ORIGIN"]
        _run(cmd)
    return EXT


def build(force: bool = False) -> None:
    build_lib(force)
    build_ext(force)


if __name__ == "__main__":
    import sys

    build(force="--force" in sys.argv)
    print(LIB)
    print(EXT)
