"""The GEMM's shared-memory operand layout is a LEGO layout: the 128-byte
swizzle as a user-defined GenP (gemm_layouts.sw128_perm) reproduces the byte
addresses TMA SWIZZLE_128B writes and the UMMA descriptors read, and the CUDA
code generator compiles it to the same arithmetic on the device."""

import numpy as np
import pytest

import paper_2505_08091_b200 as L
from paper_2505_08091_b200 import gemm_layouts as GL


def hw_sw128_byte(m, k):
    """SWIZZLE_128B for a K-major bf16 tile with 128-byte rows: inside each
    1024-byte atom, address bits [4,7) are XORed with bits [7,10)."""
    plain = m * 128 + 2 * k
    return plain ^ (((plain >> 7) & 7) << 4)


def test_swizzle_genp_is_a_bijection_and_matches_hardware():
    lay = GL.kmajor_smem_layout(128)
    assert all(line.startswith("pass") for line in str(L.validate(lay)).splitlines())
    for m in range(128):
        for k in range(64):
            assert 2 * lay.apply((m // 8, m % 8, k // 8, k % 8)) == hw_sw128_byte(m, k)


def test_swizzle_symbolic_equals_concrete():
    lay = GL.kmajor_smem_layout(64)
    idx = L.index_vars(["rh", "rl", "c", "e"], (8, 8, 8, 8))
    expr = L.apply_symbolic(lay, idx)
    for pt in [(0, 0, 0, 0), (7, 7, 7, 7), (3, 5, 2, 1), (1, 6, 7, 0), (4, 3, 5, 6)]:
        env = dict(zip(["rh", "rl", "c", "e"], pt))
        assert L.eval_expr(expr, env) == lay.apply(pt)


@pytest.mark.gpu
def test_swizzle_layout_compiles_to_the_device():
    torch = pytest.importorskip("torch")
    from paper_2505_08091_b200 import kernels as K
    lay = GL.kmajor_smem_layout(128)
    got = K.apply_map(lay).cpu().numpy()
    m, k = np.meshgrid(np.arange(128), np.arange(64), indexing="ij")
    want = np.array([hw_sw128_byte(a, b) // 2 for a, b in zip(m.ravel(), k.ravel())])
    assert np.array_equal(got, want)


def test_operand_strides_of_data_layouts():
    """Row / Col data layouts are affine with the strides TMA needs; tiled
    layouts are not (so they cannot be a tcgen05 operand as is)."""
    from paper_2505_08091_b200 import gemm_layouts as GL
    M, K = 256, 128
    row = L.parse_layout(f"GroupBy([{M},{K}]).OrderBy(Row({M},{K}))")
    col = L.parse_layout(f"GroupBy([{M},{K}]).OrderBy(Col({K},{M}))")
    assert GL.operand_strides(row) == (K, 1) and GL.operand_major(row, "A") == "row"
    assert GL.operand_strides(col) == (1, M) and GL.operand_major(col, "A") == "col"
    for i, j in ((3, 5), (200, 127), (0, 0)):
        assert row.apply((i, j)) == i * K + j and col.apply((i, j)) == i + j * M
    tiled = L.parse_layout(f"GroupBy([{M},{K}]).OrderBy(RegP([8,32,4,32],[1,3,2,4]))")
    with pytest.raises(L.UnsupportedNode):
        GL.operand_strides(tiled)


@pytest.mark.gpu
@pytest.mark.parametrize("al,bl", [("row", "row"), ("col", "row"), ("row", "col"), ("col", "col")])
def test_matmul_with_lego_data_layouts(al, bl):
    """The four matmul variants driven by LEGO Data layouts equal the string
    variants and an fp64 reference."""
    import torch
    from paper_2505_08091_b200 import kernels as K
    M, N, Kd = 512, 768, 256
    la = L.parse_layout(f"GroupBy([{M},{Kd}]).OrderBy({'Row' if al == 'row' else 'Col'}"
                        f"({M if al == 'row' else Kd},{Kd if al == 'row' else M}))")
    lb = L.parse_layout(f"GroupBy([{Kd},{N}]).OrderBy({'Row' if bl == 'row' else 'Col'}"
                        f"({Kd if bl == 'row' else N},{N if bl == 'row' else Kd}))")
    g = torch.Generator(device="cuda").manual_seed(5)
    A = torch.randn(M, Kd, device="cuda", generator=g).to(torch.bfloat16)
    B = torch.randn(Kd, N, device="cuda", generator=g).to(torch.bfloat16)
    a_buf = A.contiguous().reshape(-1) if al == "row" else A.t().contiguous().reshape(-1)
    b_buf = B.contiguous().reshape(-1) if bl == "row" else B.t().contiguous().reshape(-1)
    c = K.matmul(a_buf, b_buf, a_layout=la, b_layout=lb)
    c2 = K.matmul(a_buf.reshape((M, Kd) if al == "row" else (Kd, M)),
                  b_buf.reshape((Kd, N) if bl == "row" else (N, Kd)), a_layout=al, b_layout=bl)
    assert torch.equal(c, c2)
    ref = A.double() @ B.double()
    rel = ((c.double() - ref).abs() / ref.abs().clamp_min(1e-2 * ref.abs().max().item())).max().item()
    assert rel <= 1e-2
