"""Builds the in-tree native library libwsvd_b200.so (sm_100a CUDA kernels,
the C ABI of include/wsvd_b200.h and the C++ wsvd::decode host API).

    python -m paper_2604_02570_b200.build        # incremental, parallel

nvcc cross-compiles for sm_100a without a GPU, so this runs anywhere the
CUDA 12.9 toolkit is installed.  Objects go to paper_2604_02570_b200/_build/,
the shared library next to this file (both git-ignored, both shipped to the
GPU box by gpurun).
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
# WSVD_BUILD_TAG=x builds a variant (e.g. with WSVD_EXTRA_NVCC=-DWSVD_PIPE_DEBUG)
# into _build_x / libwsvd_b200_x.so; load it with WSVD_LIB=<that path>
_TAG = os.environ.get("WSVD_BUILD_TAG", "")
OBJ = os.path.join(PKG, "_build" + (f"_{_TAG}" if _TAG else ""))
LIB = os.path.join(PKG, "libwsvd_b200" + (f"_{_TAG}" if _TAG else "") + ".so")

NVCC = os.environ.get("NVCC", shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CUDA_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
              "--expt-relaxed-constexpr", f"-I{os.path.join(ROOT, 'include')}"]
CUDA_FLAGS += os.environ.get("WSVD_EXTRA_NVCC", "").split()  # experiment switches (-D...)
CXX_FLAGS = ["-O2", "-std=c++20", "-fPIC", "-Wall", "-Wextra", f"-I{os.path.join(ROOT, 'include')}",
             "-I/usr/local/cuda/include"]

CU_SOURCES = ["attn.cu", "attn_tc.cu", "gemm.cu", "append.cu", "step.cu", "step2.cu", "gemm_tc.cu", "dense.cu", "capi.cu"]
# host_decode.cpp (the C++ wsvd::decode drop-in) is NOT part of the library: it
# is compiled inside the reference build against the reference's own
# matrix / errors / factorize headers (oracle/Makefile target dropin)
CXX_SOURCES = ["checkpoint.cpp"]


def _stale(src: str, obj: str, deps: list[str]) -> bool:
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(d) > t for d in [src] + deps)


def _compile(cmd: list[str]) -> None:
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")


def build(verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h", ".hpp"))]
    headers += [os.path.join(ROOT, "include", "wsvd_b200.h")]
    inc_wsvd = os.path.join(ROOT, "include", "wsvd")
    if os.path.isdir(inc_wsvd):
        headers += [os.path.join(inc_wsvd, f) for f in os.listdir(inc_wsvd)]
    jobs, objs = [], []
    for f in CU_SOURCES:
        src, obj = os.path.join(CSRC, f), os.path.join(OBJ, f + ".o")
        objs.append(obj)
        if _stale(src, obj, headers):
            jobs.append([NVCC, *ARCH, *CUDA_FLAGS, "-c", src, "-o", obj])
    for f in CXX_SOURCES:
        src, obj = os.path.join(CSRC, f), os.path.join(OBJ, f + ".o")
        if not os.path.exists(src):
            continue
        objs.append(obj)
        if _stale(src, obj, headers):
            jobs.append(["g++", *CXX_FLAGS, "-c", src, "-o", obj])
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        for cmd in jobs:
            if verbose:
                print(" ".join(cmd))
        list(ex.map(_compile, jobs))
    if jobs or not os.path.exists(LIB) or any(os.path.getmtime(o) > os.path.getmtime(LIB) for o in objs):
        _compile([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", LIB, *objs, "-ldl", "-lpthread", "-lrt"])
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
