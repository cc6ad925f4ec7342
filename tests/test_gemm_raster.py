"""The GEMM's CTA tile raster is a LEGO layout.

CPU: the grouped raster written as a user GenP over the (m-block, n-block)
grid agrees with ``raster_layout`` (GroupBy([MB/G, NB, G]).OrderBy(Row)) when
G divides MB, and is a bijection with its inverse otherwise (tail group).
GPU: the tile order the kernels evaluate (``tile_coords`` in
csrc/gemm_tcgen05.cu, dumped by ``lego_gemm_raster``) equals the LEGO
layout's inverse map computed by the generated index-map kernel
(``kernels.inv_map``), for the group sizes both GEMM kernels pass.
"""

import itertools

import pytest

import paper_2505_08091_b200 as L
from paper_2505_08091_b200 import gemm_layouts as GL


@pytest.mark.parametrize("mb,nb,g", [(64, 32, 16), (16, 4, 16), (32, 7, 8), (64, 32, 32)])
def test_grouped_perm_matches_raster_layout(mb, nb, g):
    perm = GL.grouped_raster_perm(mb, nb, g)
    blk = GL.raster_layout(mb, nb, g)
    for t in range(mb * nb):
        grp, n, m_in = blk.inv(t)
        assert perm.inv(t) == (grp * g + m_in, n)
        assert perm.apply((grp * g + m_in, n)) == t


@pytest.mark.parametrize("mb,nb,g", [(20, 3, 16), (5, 4, 2), (33, 2, 8), (7, 9, 1)])
def test_grouped_perm_with_tail_is_a_bijection(mb, nb, g):
    perm = GL.grouped_raster_perm(mb, nb, g)
    lay = L.GroupBy([mb, nb]).order_by(perm)
    seen = {perm.inv(t) for t in range(mb * nb)}
    assert seen == set(itertools.product(range(mb), range(nb)))
    t_var = L.Var("t", L.VarRange(0, mb * nb))
    m_e, n_e = L.inv_symbolic(lay, t_var)
    for t in range(mb * nb):
        assert (L.eval_expr(m_e, {"t": t}), L.eval_expr(n_e, {"t": t})) == perm.inv(t)


def _lego_raster(mb, nb, g, batch):
    """GroupBy([batch, mb, nb]).OrderBy(Row(batch), grouped raster): tile t -> (b, m, n)."""
    perm = GL.grouped_raster_perm(mb, nb, g) if g else L.RegP([mb, nb], [1, 2])
    return L.GroupBy([batch, mb, nb]).order_by(L.RegP([batch], [1]), perm)


@pytest.mark.gpu
@pytest.mark.parametrize("mb,nb,batch,g", [(64, 32, 1, 32), (64, 32, 2, 16), (32, 16, 1, 0), (20, 3, 2, 16),
                                           (33, 2, 3, 8), (16, 16, 1, 1), (32, 16, 8, 16)])
def test_device_raster_is_the_lego_inverse(mb, nb, batch, g):
    torch = pytest.importorskip("torch")
    from paper_2505_08091_b200 import kernels as K
    dev = K.gemm_raster(mb, nb, batch, g).long()
    x = K.inv_map(_lego_raster(mb, nb, g, batch), dtype=torch.int64)
    want = torch.stack([x // (mb * nb), (x // nb) % mb, x % nb], dim=1)
    assert torch.equal(dev, want)


@pytest.mark.gpu
def test_default_rasters_of_cfg5():
    """8192^3 (cfg5): the pair kernel's 32 x 16 tiles of 256 x 512 with G/2,
    the single-CTA kernel's 64 x 32 tiles of 128 x 256 with G."""
    torch = pytest.importorskip("torch")
    from paper_2505_08091_b200 import kernels as K
    G = K.GEMM_RASTER_GROUP
    for mb, nb, g in ((8192 // 256, 8192 // 512, G // 2), (8192 // 128, 8192 // 256, G)):
        dev = K.gemm_raster(mb, nb, 1, g).long()
        x = K.inv_map(_lego_raster(mb, nb, g, 1), dtype=torch.int64)
        assert torch.equal(dev[:, 1] * nb + dev[:, 2], x)
