"""The C ABI: the in-tree library loads without a GPU, exports every symbol
include/lego_b200.h declares, and the JIT path (NVRTC, no GPU needed)
compiles generated programs for sm_100a.  No compute calls here."""

import ctypes
import os
import re

import pytest

import paper_2505_08091_b200 as L
from paper_2505_08091_b200 import kernels as K
from paper_2505_08091_b200 import runtime as R

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "lego_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(lego_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(R.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 14
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) <= set(R.SIGS), set(syms) - set(R.SIGS)


def test_abi_version_and_error_channel():
    lib = R.lib()
    assert lib.lego_abi_version() == 1
    assert isinstance(lib.lego_last_error(), bytes)


def test_null_arguments_fail_cleanly():
    lib = R.lib()
    st = lib.lego_remap(None, None, None, 1, 0, 0, None)
    assert st == 8 and b"not a remap program" in lib.lego_last_error()
    st = lib.lego_softmax_f32(None, None, 4, 3, None)
    assert st == 8 and b"null buffer" in lib.lego_last_error()
    st = lib.lego_softmax_f32(None, None, 4, 0, None)
    assert st == 3 and b"bad softmax shape" in lib.lego_last_error()
    with pytest.raises(L.ShapeMismatch):
        R.check(lib.lego_gemm_bf16(None, None, None, 100, 250, 64, 1, 1, None))   # N % 8
    # NW: argument checks run before any CUDA call (offset-score range, alignment)
    buf = ctypes.create_string_buffer(64 + 16)
    aligned = (ctypes.addressof(buf) + 15) & ~15
    st = lib.lego_nw_i32(aligned, aligned, 16384, 40000, 1, None)
    assert st == 8 and b"penalty" in lib.lego_last_error()
    st = lib.lego_nw_i32(aligned + 4, aligned, 16, 10, 1, None)
    assert st == 8 and b"16-byte aligned" in lib.lego_last_error()
    assert lib.lego_nw_i32(aligned, aligned, 16, 10, 0, None) == 0     # empty batch
    # NW column band (multi-GPU single alignment): band and edge arguments
    st = lib.lego_nw_band_i32(aligned, aligned, 300, 10, 1, 2, 4, aligned, None, 0, 0, None)
    assert st == 3 and b"strip band" in lib.lego_last_error()         # 300 columns = 3 strips
    st = lib.lego_nw_band_i32(aligned, aligned, 300, 10, 1, 1, 3, aligned, None, 0, 0, None)
    assert st == 8 and b"left_words" in lib.lego_last_error()         # band after strip 0 needs the left edge
    st = lib.lego_nw_band_i32(aligned, aligned, 300, 10, 1, 0, 3, aligned + 4, None, 0, 0, None)
    assert st == 8 and b"16-byte aligned" in lib.lego_last_error()
    st = lib.lego_nw_band_i32(aligned, aligned, 300, 10, 1, 1, 3, aligned, aligned, 8, 0, None)
    assert st == 8 and b"left_batch_stride" in lib.lego_last_error()


@pytest.mark.parametrize("dsl", [
    "GroupBy([4096,4096]).OrderBy(RegP([128,32,128,32],[1,3,2,4]))",
    "GroupBy([64,64]).OrderBy(Col(64,64))",
    "GroupBy([64,64]).OrderBy(GenP([64,64], antidiag))",
    "ExpandBy([30,28],[32,32],GroupBy([32,32]).OrderBy(RegP([2,16,2,16],[1,3,2,4])))",
    "GroupBy([6,6]).OrderBy(RegP([2,3,2,3],[1,3,2,4])).OrderBy(RegP([2,2],[2,1]), GenP([3,3], antidiag))",
])
def test_generated_programs_compile_for_sm100a(dsl):
    g = L.parse_layout(dsl)
    cubin = R.compile_cubin(K.index_map_source(g)[0])
    assert cubin[:4] == b"\x7fELF"
    for e in (2, 4):
        plan = K.plan_remap(None, g, e) if g.size % (16 // e) == 0 else None
        if plan is not None:
            assert R.compile_cubin(plan.source)[:4] == b"\x7fELF"


def test_kernel_selection():
    col = L.parse_layout("GroupBy([16384,16384]).OrderBy(Col(16384,16384))")
    assert "transpose" in repr(K.plan_remap(None, col, 2))
    tiled = L.parse_layout("GroupBy([4096,4096]).OrderBy(RegP([128,32,128,32],[1,3,2,4]))")
    p = K.plan_remap(None, tiled, 4)
    assert "gather" in repr(p) and p.contig
    ad = L.parse_layout("GroupBy([16384,16384]).OrderBy(GenP([16384,16384], antidiag))")
    assert "band" in repr(K.plan_remap(None, ad, 4))
    assert "band" in repr(K.plan_remap(ad, None, 4))
