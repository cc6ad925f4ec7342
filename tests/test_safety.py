"""Argument checks and write-safety gates of the bulk operations (the C ABI
takes bare pointers, so the Python boundary validates what it passes).

* caller-provided ``out`` tensors: dtype, device, contiguity, size;
* ``inv_map`` of an injective-mode layout raises like the reference's
  ``GroupBy.inv`` (layout.py:321-322);
* ``gemm`` operands: device, batch dims;
* stores through user GenPs above the reference's 4096-point trust bound
  (layout.py:718-719) are proven injective / bijective on the device once
  per program before the first launch, and refused otherwise.
"""

import pytest

import paper_2505_08091_b200 as L

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2505_08091_b200 import kernels as K  # noqa: E402


def _even(n, collide=False):
    f = (lambda i: (i[0] // 2) * 4) if collide else (lambda i: i[0] * 2)
    return L.GenP((n,), L.PermFn(f, f), None, name=None)


def test_out_checks():
    g = L.parse_layout("GroupBy([64,64]).OrderBy(Col(64,64))")
    x = torch.arange(64 * 64, dtype=torch.int32, device="cuda")
    for bad in (torch.empty(64 * 64 - 1, dtype=torch.int32, device="cuda"),          # too small
                torch.empty(64 * 64, dtype=torch.float32, device="cuda"),            # dtype
                torch.empty(2 * 64 * 64, dtype=torch.int32, device="cuda")[::2],     # strided
                torch.empty(64 * 64, dtype=torch.int32)):                            # host
        with pytest.raises(L.ShapeMismatch):
            K.remap(x, None, g, out=bad)
    with pytest.raises(L.ShapeMismatch):
        K.apply_map(g, out=torch.empty(10, dtype=torch.int32, device="cuda"))
    with pytest.raises(L.ShapeMismatch):
        K.inv_map(g, out=torch.empty(64 * 64, dtype=torch.float32, device="cuda"))
    with pytest.raises(L.OutOfBounds):
        K.apply_map(g, first=10, count=64 * 64)
    y = torch.randn(4, 1024, device="cuda")
    with pytest.raises(L.ShapeMismatch):
        K.softmax(y, out=torch.empty(4, 1000, device="cuda"))
    sim = torch.zeros(8, 8, dtype=torch.int32, device="cuda")
    with pytest.raises(L.ShapeMismatch):
        K.nw_score(sim, 1, out=torch.empty(8, 8, dtype=torch.int32, device="cuda"))


def test_inv_map_of_injective_layout_raises():
    lay = L.GroupBy([4096], orders=(L.OrderBy(_even(4096)),), injective=True)
    assert torch.equal(K.apply_map(lay).cpu(), torch.arange(4096, dtype=torch.int32) * 2)
    with pytest.raises(L.LegoError):
        K.inv_map(lay)


def test_gemm_operand_checks():
    a = torch.zeros(2, 128, 64, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(L.ShapeMismatch):
        K.gemm(a, torch.zeros(2, 256, 64, dtype=torch.bfloat16))                 # host b
    with pytest.raises(L.ShapeMismatch):
        K.gemm(a, torch.zeros(256, 64, dtype=torch.bfloat16, device="cuda"))    # batch dims differ
    with pytest.raises(L.ShapeMismatch):
        K.gemm(a, torch.zeros(2, 256, 64, dtype=torch.bfloat16, device="cuda"),
               out=torch.empty(2, 128, 255, dtype=torch.bfloat16, device="cuda"))


def test_scatter_through_user_genp_is_gated():
    n = 1 << 16                                                   # > the 4096-point trust bound
    ok = L.GroupBy([n], orders=(L.OrderBy(_even(n)),), injective=True)
    x = torch.arange(n, dtype=torch.int32, device="cuda")
    prog_before = K.LAUNCHES[0]
    out = K.remap(x, None, ok)
    assert K.LAUNCHES[0] - prog_before == 3                     # histogram + check + scatter
    assert torch.equal(out[::2], x) and not out[1::2].any()
    prog_before = K.LAUNCHES[0]
    K.remap(x, None, ok, out=out, fill=0)                        # proven once per program
    assert K.LAUNCHES[0] - prog_before == 1
    bad = L.GroupBy([n], orders=(L.OrderBy(_even(n, collide=True)),), injective=True)
    with pytest.raises(L.BijectivityViolation):
        K.remap(x, None, bad)
    assert K.check_injective(ok) and not K.check_injective(bad)


def test_small_user_genp_is_trusted_like_the_reference():
    n = 4096                                                     # validate() enumerates these
    lay = L.GroupBy([n], orders=(L.OrderBy(_even(n)),), injective=True)
    before = K.LAUNCHES[0]
    K.remap(torch.arange(n, dtype=torch.int32, device="cuda"), None, lay)
    assert K.LAUNCHES[0] - before == 1
