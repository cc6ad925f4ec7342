"""The Needleman-Wunsch wavefront driven by LEGO layouts (paper_2505_08091_b200.nw).

CPU: the layout form and its meaning (position = T(a,b)*H*128 + I(r,c), the
reference GroupBy/OrderBy semantics), the host proofs (topological tile
order, row-preserving 16-byte cell order) accepting valid and rejecting
invalid layouts, and NVRTC compilation of the generated programs.
GPU: every layout bit-exact against the C DP (oracle.nw) at
n in {1, 7, 100, 1024, 16384}, with built-in and user-defined tile orders
(antidiag, skew, Morton, column-major) and user-defined cell orders.
"""

import numpy as np
import pytest

import paper_2505_08091_b200 as L
from paper_2505_08091_b200 import nw
from nw_perms import morton_order, nw_test_layouts, rotate_cells, skew_order, xor_cells

SIZES = [1, 7, 100, 1024, 16384]


@pytest.mark.parametrize("n,h,order", [(100, 32, None), (300, 64, "col"), (256, 128, "antidiag"),
                                       (512, 128, "skew"), (512, 64, "morton")])
def test_layout_meaning(n, h, order):
    """L.apply((i, j)) == T(i//H, j//128) * H*128 + I(i%H, j%128) on sampled cells."""
    nr, nc = -(-n // h), -(-n // 128)
    t = {"skew": lambda: skew_order(nr, nc), "morton": lambda: morton_order(nr)}.get(order, lambda: order)()
    if order == "morton" and nr != nc:
        pytest.skip("morton needs a square grid")
    lay = nw.nw_layout(n, tile_rows=h, tile_order=t, cell_order=rotate_cells(h))
    parts = nw.nw_parts(lay, n)
    rng = np.random.default_rng(n)
    for i, j in rng.integers(0, n, size=(200, 2)):
        i, j = int(i), int(j)
        want = parts.tiles.apply((i // h, j // 128)) * h * 128 + parts.cells.apply((i % h, j % 128))
        assert lay.apply((i, j)) == want


def test_default_layout_is_strips():
    lay = nw.nw_layout(1000)
    parts = nw.nw_parts(lay, 1000)
    assert (parts.h, parts.nr, parts.nc) == (1000, 1, 8)
    assert nw.slot_identity(parts)
    # the DSL spelling parses to the same layout
    assert L.parse_layout("GroupBy([1000,1024]).OrderBy(RegP([1,1000,8,128],[1,3,2,4]))") == lay


@pytest.mark.parametrize("n", SIZES)
def test_host_proofs_accept_test_layouts(n):
    for name, lay in nw_test_layouts(n):
        parts = nw.nw_parts(lay, n)
        nw.host_check_tile_order(parts)
        nw.host_check_cell_order(parts)


def _rev(shape):
    return L.reverse_perm(shape)


@pytest.mark.parametrize("order", ["rev", "transposed-col-of-rows", "swap"])
def test_host_proof_rejects_non_topological_orders(order):
    n, h = 512, 128
    nr = nc = 4
    if order == "rev":
        t = _rev((nr, nc))
    elif order == "transposed-col-of-rows":
        # rows bottom-up: tile (a, b) -> (nr-1-a)*nc + b
        t = L.GenP((nr, nc), L.PermFn(lambda ix: (nr - 1 - ix[0]) * nc + ix[1],
                                      lambda ix: ((nr - 1) - ix[0]) * nc + ix[1]),
                   L.PermFn(lambda f: (nr - 1 - f // nc, f % nc), lambda f: ((nr - 1) - f // nc, f % nc)))
    else:
        # row-major with tiles (0, 1) and (1, 0) swapped is still topological; (0,0)<->(0,1) is not
        def fwd(ix):
            x = ix[0] * nc + ix[1]
            return {0: 1, 1: 0}.get(x, x)
        t = L.GenP((nr, nc), L.PermFn(fwd, fwd), L.PermFn(lambda f: divmod({0: 1, 1: 0}.get(f, f), nc),
                                                         lambda f: divmod({0: 1, 1: 0}.get(f, f), nc)))
    parts = nw.nw_parts(nw.nw_layout(n, tile_rows=h, tile_order=t), n)
    with pytest.raises(L.UnsupportedNode):
        nw.host_check_tile_order(parts)


def test_host_proof_rejects_bad_cell_orders():
    n, h = 256, 64
    for cells in (L.RegP([h, 128], [2, 1]),                      # column-major: moves cells across rows
                  L.reverse_perm((h, 128))):                      # reverses rows and breaks lane groups
        parts = nw.nw_parts(nw.nw_layout(n, tile_rows=h, cell_order=cells), n)
        with pytest.raises(L.UnsupportedNode):
            nw.host_check_cell_order(parts)
    # per-row reversal of the 4-column groups keeps rows and vectors: accepted
    def fwd(ix):
        r, c = ix
        return r * 128 + 4 * (31 - c // 4) + c % 4
    ok = L.GenP((h, 128), L.PermFn(fwd, fwd), None)
    nw.host_check_cell_order(nw.nw_parts(nw.nw_layout(n, tile_rows=h, cell_order=ok), n))


def test_rejects_other_forms():
    with pytest.raises(L.UnsupportedNode):
        nw.nw_parts(L.parse_layout("GroupBy([256,256]).OrderBy(Col(256,256))"), 256)
    with pytest.raises(L.UnsupportedNode):       # 64-column tiles
        nw.nw_parts(L.parse_layout("GroupBy([256,256]).OrderBy(RegP([2,128,4,64],[1,3,2,4]))"), 256)
    with pytest.raises(L.ShapeMismatch):         # grid does not match n
        nw.nw_parts(nw.nw_layout(256, tile_rows=64), 100)
    with pytest.raises(L.UnsupportedNode):       # tile rows not a multiple of 32
        nw.nw_parts(nw.nw_layout(100, tile_rows=20), 100)


@pytest.mark.parametrize("n", [7, 1024])
def test_programs_compile(n):
    from paper_2505_08091_b200 import runtime as R
    for name, lay in nw_test_layouts(n):
        src, info, defines = nw.program_source(nw.nw_parts(lay, n))
        assert info.kind == nw.KIND_NW and info.smem_bytes == nw.SMEM_BYTES
        if "+" in name:
            assert defines["NW_GEN_TILES"] or defines["NW_GEN_SLOTS"], name
        assert len(R.compile_cubin(src)) > 1000


# ---------------------------------------------------------------------------
# GPU: bit-exact against the C DP
# ---------------------------------------------------------------------------

def _sim(n, batch, seed):
    rng = np.random.default_rng(seed)
    return rng.integers(-10, 11, size=(batch, n, n), dtype=np.int32)


@pytest.mark.gpu
@pytest.mark.parametrize("n", SIZES)
def test_nw_layouts_bit_exact(n):
    torch = pytest.importorskip("torch")
    from paper_2505_08091_b200 import kernels as K
    from oracle import oracle as O
    batch = 1 if n >= 1024 else 2
    sim = _sim(n, batch, 4 + n)
    want = np.stack([O.nw(sim[b], 10) for b in range(batch)])
    dsim = torch.from_numpy(sim).cuda()
    names = []
    for name, lay in nw_test_layouts(n):
        got = K.nw_score(dsim, 10, layout=lay).cpu().numpy()
        assert np.array_equal(got, want), (n, name, np.argwhere(got != want)[:5])
        names.append(name)
    assert len(names) >= 2


@pytest.mark.gpu
def test_nw_layout_rejected_before_launch():
    torch = pytest.importorskip("torch")
    from paper_2505_08091_b200 import kernels as K
    sim = torch.zeros(512, 512, dtype=torch.int32, device="cuda")
    lay = nw.nw_layout(512, tile_rows=128, tile_order=_rev((4, 4)))
    with pytest.raises(L.UnsupportedNode):
        K.nw_score(sim, 10, layout=lay)


@pytest.mark.gpu
def test_nw_layout_tiles_batch_and_penalties():
    torch = pytest.importorskip("torch")
    from paper_2505_08091_b200 import kernels as K
    from oracle import oracle as O
    n = 640
    sim = _sim(n, 3, 11)
    lay = nw.nw_layout(n, tile_rows=64, tile_order=skew_order(10, 5), cell_order=xor_cells(64))
    for p in (0, 3, -2):
        got = K.nw_score(torch.from_numpy(sim).cuda(), p, layout=lay).cpu().numpy()
        for b in range(3):
            assert np.array_equal(got[b], O.nw(sim[b], p)), (p, b)


def test_default_strips_use_the_library_kernel():
    """Tuning defines (skew, readiness cadence) alone do not require a generated program."""
    src, info, d = nw.program_source(nw.nw_parts(nw.nw_layout(1000), 1000))
    assert d["NW_SKEW"] == 1 and not nw.needs_program(d)
    src, info, d = nw.program_source(nw.nw_parts(nw.nw_layout(4096, tile_rows=2048), 4096))
    assert d["NW_SKEW"] == 2 and d["NW_GRP"] == 4 and nw.needs_program(d)
