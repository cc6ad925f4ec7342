"""The GEMM's CTA raster is a LEGO layout: its inverse, derived symbolically,
is exactly the arithmetic gemm_tcgen05.cu evaluates (Raster::coords)."""

import itertools

import paper_2505_08091_b200 as L

G = 16  # GROUP_M in gemm_tcgen05.cu


def kernel_coords(t, mb, nb):
    """Python mirror of Raster::coords in csrc/gemm_tcgen05.cu."""
    per_batch = mb * nb
    b, r = divmod(t, per_batch)
    full = (mb // G) * G
    g_tiles = G * nb
    if r < (full // G) * g_tiles or full == mb:
        g, rem = divmod(r, g_tiles)
        n, m_in = divmod(rem, G)
        return b, g * G + m_in, n
    tail = mb - full
    rem = r - (full // G) * g_tiles
    n, m_in = divmod(rem, tail)
    return b, full + m_in, n


def test_raster_is_the_lego_layout_inverse():
    for mb, nb in ((64, 32), (16, 4), (32, 7)):
        blk = L.parse_layout(f"GroupBy([{mb // G},{nb},{G}]).OrderBy(Row({mb // G},{nb},{G}))")
        t = L.Var("t", L.VarRange(0, mb * nb))
        g, n, m_in = L.inv_symbolic(blk, t)
        for tv in range(mb * nb):
            env = {"t": tv}
            want = (0, L.eval_expr(g, env) * G + L.eval_expr(m_in, env), L.eval_expr(n, env))
            assert kernel_coords(tv, mb, nb) == want


def test_raster_with_tail_group_is_a_bijection():
    for mb, nb, batch in ((20, 3, 2), (5, 4, 1), (33, 2, 3)):
        seen = {kernel_coords(t, mb, nb) for t in range(mb * nb * batch)}
        assert seen == set(itertools.product(range(batch), range(mb), range(nb)))
