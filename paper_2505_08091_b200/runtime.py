"""ctypes binding of ``liblego_b200.so`` (the C ABI in ``include/lego_b200.h``).

The library is built in-tree by :mod:`.build`.  If it is missing the
backend raises :class:`BackendUnavailable` -- there is no CPU fallback.
Status codes map back onto the reference exception classes
(``pkg/src/lego/errors.py``), messages come from ``lego_last_error``.
"""

from __future__ import annotations

import ctypes
import hashlib
import os
import threading
from typing import Optional

from .errors import (
    ArityMismatch,
    BackendUnavailable,
    BijectivityViolation,
    CudaError,
    LegoError,
    OutOfBounds,
    ShapeMismatch,
    UnsupportedNode,
)

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LEGO_B200_LIB") or os.path.join(PKG, "liblego_b200.so")   # override: A/B builds
CACHE_DIR = os.environ.get("LEGO_B200_KCACHE", os.path.join(PKG, "kcache"))
ARCH = "sm_100a"

_STATUS = {
    1: ArityMismatch,
    2: OutOfBounds,
    3: ShapeMismatch,
    4: UnsupportedNode,
    5: CudaError,
    6: CudaError,
    7: BijectivityViolation,
    8: LegoError,
}


class ProgramInfo(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("elem_bytes", ctypes.c_int32), ("n", ctypes.c_int64),
                ("units", ctypes.c_int64), ("unit_threads", ctypes.c_int32),
                ("block", ctypes.c_int32), ("smem_bytes", ctypes.c_int32),
                ("reserved", ctypes.c_int32)]


KIND_INDEX_MAP, KIND_GATHER, KIND_TRANSPOSE, KIND_BAND, KIND_SCATTER, KIND_STAGED, KIND_NW, KIND_SOFTMAX = 0, 1, 2, 3, 4, 5, 6, 7
# lego_program_info.reserved flags (include/lego_b200.h): element-aligned buffers suffice
ALIGN_SRC_FREE, ALIGN_DST_FREE = 1, 2
FILL_FUSED, FILL_PASS = 4, 8

_lib = None
_lock = threading.Lock()

VP = ctypes.c_void_p
I32 = ctypes.c_int32
I64 = ctypes.c_int64
SIGS = {
    "lego_abi_version": ([], I32),
    "lego_last_error": ([], ctypes.c_char_p),
    "lego_device_info": ([I32, ctypes.POINTER(I32), ctypes.POINTER(I64), ctypes.POINTER(I32),
                          ctypes.POINTER(I32)], I32),
    "lego_nvrtc_compile": ([ctypes.c_char_p, ctypes.c_size_t, ctypes.c_char_p,
                            ctypes.POINTER(VP), ctypes.POINTER(ctypes.c_size_t),
                            ctypes.c_char_p, ctypes.c_size_t], I32),
    "lego_free": ([VP], None),
    "lego_program_load": ([VP, ctypes.c_size_t, ctypes.POINTER(ProgramInfo), ctypes.POINTER(VP)], I32),
    "lego_program_release": ([VP], None),
    "lego_module_load": ([VP, ctypes.c_size_t, ctypes.POINTER(VP)], I32),
    "lego_module_release": ([VP], None),
    "lego_module_launch": ([VP, ctypes.c_char_p, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32,
                            ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32,
                            ctypes.POINTER(VP), VP], I32),
    "lego_apply_map": ([VP, VP, I32, I64, I64, VP], I32),
    "lego_inv_map": ([VP, VP, I32, I64, I64, VP], I32),
    "lego_check_bijective": ([VP, VP, ctypes.POINTER(I64), VP], I32),
    "lego_check_injective": ([VP, VP, ctypes.POINTER(I64), VP], I32),
    "lego_remap": ([VP, VP, VP, I64, I64, I64, VP], I32),
    "lego_remap_fill": ([VP, VP, VP, I64, I64, I64, VP, VP], I32),
    "lego_softmax_f32": ([VP, VP, I64, I64, VP], I32),
    "lego_nw_i32": ([VP, VP, I64, I32, I64, VP], I32),
    "lego_nw_run": ([VP, VP, VP, I64, I32, I64, VP], I32),
    "lego_nw_band_i32": ([VP, VP, I64, I32, I64, I64, I64, VP, VP, I64, I32, VP], I32),
    "lego_softmax_run": ([VP, VP, VP, I64, I64, VP], I32),
    "lego_softmax_offsets": ([VP, VP, I64, VP], I32),
    "lego_gemm_raster": ([VP, I64, I64, I64, I32, VP], I32),
    "lego_gemm_bf16": ([VP, VP, VP, I64, I64, I64, I64, I32, VP], I32),
    "lego_gemm_bf16_ex": ([VP, VP, VP, I64, I64, I64, I64, I32, I32, I32, VP], I32),
}


def lib():
    """Load (once) and type the native library; raise if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise BackendUnavailable(
                    f"{LIB_PATH} is missing; build it with `python -m paper_2505_08091_b200.build` "
                    "(there is no CPU fallback)")
            handle = ctypes.CDLL(LIB_PATH)
            for name, (args, res) in SIGS.items():
                fn = getattr(handle, name)
                fn.argtypes = args
                fn.restype = res
            if handle.lego_abi_version() != 1:
                raise BackendUnavailable("liblego_b200.so ABI version mismatch")
            _lib = handle
    return _lib


def check(status: int, what: str = ""):
    if status == 0:
        return
    msg = lib().lego_last_error().decode(errors="replace")
    exc = _STATUS.get(status, LegoError)
    raise exc(f"{what}: {msg}" if what else msg)


def device_info(device: int = 0):
    sm, l2, ma, mi = I32(), I64(), I32(), I32()
    check(lib().lego_device_info(device, ctypes.byref(sm), ctypes.byref(l2), ctypes.byref(ma),
                                 ctypes.byref(mi)), "lego_device_info")
    return {"sm_count": sm.value, "l2_bytes": l2.value, "cc": (ma.value, mi.value)}


def cubin_path(source: str) -> str:
    """Cache file of a program text (SHA-256 of arch + source)."""
    key = hashlib.sha256((ARCH + "\0" + source).encode()).hexdigest()[:32]
    return os.path.join(CACHE_DIR, key + ".cubin")


def compile_cubin(source: str) -> bytes:
    """NVRTC-compile a generated program for sm_100a, cached on disk by the
    SHA-256 of its text (the cache travels with the repo snapshot)."""
    path = cubin_path(source)
    if os.path.exists(path):
        with open(path, "rb") as fh:
            return fh.read()
    out, n = VP(), ctypes.c_size_t()
    log = ctypes.create_string_buffer(1 << 16)
    src = source.encode()
    check(lib().lego_nvrtc_compile(src, len(src), ARCH.encode(), ctypes.byref(out), ctypes.byref(n),
                                   log, len(log)), "lego_nvrtc_compile")
    try:
        data = ctypes.string_at(out, n.value)
    finally:
        lib().lego_free(out)
    try:
        os.makedirs(CACHE_DIR, exist_ok=True)
        tmp = f"{path}.{os.getpid()}.tmp"
        with open(tmp, "wb") as fh:
            fh.write(data)
        os.replace(tmp, path)
    except OSError:
        pass
    return data


class Program:
    """A loaded generated program (owns the module; released on GC)."""

    def __init__(self, cubin: bytes, info: ProgramInfo, source: str = ""):
        self.info = info
        self.source = source
        self._cubin = ctypes.create_string_buffer(cubin, len(cubin))
        h = VP()
        check(lib().lego_program_load(self._cubin, len(cubin), ctypes.byref(info), ctypes.byref(h)),
              "lego_program_load")
        self.handle = h

    def __del__(self):
        h = getattr(self, "handle", None)
        if h and _lib is not None:
            try:
                _lib.lego_program_release(h)
            except Exception:  # noqa: BLE001 - interpreter teardown
                pass
            self.handle = None


class Module:
    """A user kernel module (e.g. an instantiated LEGO ``.cu`` template)
    compiled for sm_100a; ``launch`` runs one of its ``extern "C"`` kernels."""

    def __init__(self, cubin: bytes):
        self._cubin = ctypes.create_string_buffer(cubin, len(cubin))
        h = VP()
        check(lib().lego_module_load(self._cubin, len(cubin), ctypes.byref(h)), "lego_module_load")
        self.handle = h

    def launch(self, kernel: str, grid, block, args, *, smem: int = 0, stream=None):
        """``args``: ctypes values (c_void_p for device pointers, c_int64, ...)."""
        grid = tuple(grid) + (1,) * (3 - len(tuple(grid)))
        block = tuple(block) + (1,) * (3 - len(tuple(block)))
        ptrs = (VP * max(1, len(args)))(*[ctypes.cast(ctypes.pointer(a), VP) for a in args])
        check(lib().lego_module_launch(self.handle, kernel.encode(), *grid, *block, smem, ptrs,
                                       stream_handle(stream)), f"lego_module_launch({kernel})")

    def __del__(self):
        h = getattr(self, "handle", None)
        if h and _lib is not None:
            try:
                _lib.lego_module_release(h)
            except Exception:  # noqa: BLE001 - interpreter teardown
                pass
            self.handle = None


def stream_handle(stream=None) -> Optional[int]:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream
