"""Build liblego_b200.so in-tree for sm_100a (``nvcc`` cross-compiles; no GPU needed).

    python -m paper_2505_08091_b200.build [--force]

The library is the C-ABI of ``include/lego_b200.h``: the runtime (NVRTC JIT
of generated layout kernels, program loading, launches) plus the fixed
kernels (softmax, Needleman-Wunsch wavefront, tcgen05 GEMM).
"""

from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "liblego_b200.so")
SOURCES = ["lego_runtime.cu", "softmax.cu", "wavefront.cu", "gemm_tcgen05.cu"]
DEPS = ["lego_common.h", "lego_index.cuh", "remap_kernels.cuh", "nw_kernels.cuh", "softmax_kernels.cuh", "../../include/lego_b200.h"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    return "nvcc"


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    for f in SOURCES + DEPS:
        p = os.path.join(CSRC, f)
        if os.path.exists(p) and os.path.getmtime(p) > t:
            return True
    return False


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    objs = []
    build_dir = os.path.join(PKG, "..", "build", "obj")
    os.makedirs(build_dir, exist_ok=True)
    only = [x for x in os.environ.get("LEGO_BUILD_ONLY", "").split(",") if x]
    for src in SOURCES:
        path = os.path.join(CSRC, src)
        obj = os.path.join(build_dir, src.replace(".cu", ".o"))
        if only and src not in only and os.path.exists(obj):
            objs.append(obj)           # development: reuse the other objects as built
            continue
        cmd = [nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
               "-Xptxas", "-v" if verbose else "-O3", *os.environ.get("LEGO_NVCC_FLAGS", "").split(),
               "-c", path, "-o", obj]
        subprocess.check_call(cmd)
        objs.append(obj)
    tmp = LIB + ".tmp"
    subprocess.check_call([nvcc(), *ARCH, "-shared", "-o", tmp, *objs, "-ldl", "-lpthread"])
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
