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
