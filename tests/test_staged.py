"""Box-staged gathers (paper_2505_08091_b200/staging.py, LEGO_KIND 5).

CPU: the planner's decomposition g(q*B + r) == base(q) + row(r)*SX + col(r)
is checked against the C oracle's inverse map at every position, and the
vectorised evaluator against the exact one.  GPU: the staged kernel against
the oracle, bit-exact, for 1/2/4/8-byte elements, batches, unaligned sources
and the full-size SURVEY f1 chain."""

import numpy as np
import pytest

from oracle import oracle as O

import paper_2505_08091_b200 as L
from paper_2505_08091_b200 import kernels as K, lower, runtime, staging
from paper_2505_08091_b200.expr import eval_expr

STAGED = [
    # multi-stage chain, in-tile anti-diagonal GenP (SURVEY f1 / Eq. (2) shape)
    "GroupBy([512,512]).OrderBy(RegP([16,32,16,32],[1,3,2,4])).OrderBy(RegP([16,16],[2,1]), GenP([32,32], antidiag))",
    # tiles in column order, in-tile reversal
    "GroupBy([1024,256]).OrderBy(RegP([16,64,4,64],[1,3,2,4])).OrderBy(RegP([16,4],[1,2]), GenP([64,64], rev2d))",
    # 64 x 64 anti-diagonal tiles of a 256 x 256 matrix (f1 at a small size)
    "GroupBy([256,256]).OrderBy(RegP([4,64,4,64],[1,3,2,4])).OrderBy(RegP([4,4],[2,1]), GenP([64,64], antidiag))",
]


def _offsets_hold(text, elem):
    g = L.parse_layout(text)
    spec = O.parse(text)
    f, gx, n_dst, n_src = lower.gather_expr(None, g)
    bp = staging.box_plan(gx, f, n_dst, n_src, elem)
    assert bp is not None, text
    B = bp.block
    inv = O.inv_range(spec)                     # source (row-major) index of dst position f
    q = np.arange(n_dst, dtype=np.int64) // B
    base = staging.eval_vec(bp.base, {"q": q})
    off = np.tile(bp.offsets.astype(np.int64), n_dst // B)
    got = base + (off // bp.pitch) * bp.sx + off % bp.pitch
    np.testing.assert_array_equal(got, inv)
    # every box cell is read exactly once per block
    rows, cols = bp.offsets // bp.pitch, bp.offsets % bp.pitch
    assert rows.max() < bp.rows and cols.max() < bp.cols
    assert len(np.unique(bp.offsets)) == bp.rows * bp.cols == B
    return bp


@pytest.mark.parametrize("text", STAGED)
@pytest.mark.parametrize("elem", [1, 2, 4, 8])
def test_box_decomposition_matches_oracle(text, elem):
    bp = _offsets_hold(text, elem)
    assert bp.rows * bp.pitch * elem <= staging.BOX_SMEM
    p = K.plan_remap(None, L.parse_layout(text), elem)
    assert p.kind == runtime.KIND_STAGED, p
    # the mirrored direction (layout -> row-major) stages source blocks
    p = K.plan_remap(L.parse_layout(text), None, elem)
    assert p.kind in (runtime.KIND_STAGED, runtime.KIND_TRANSPOSE), p


@pytest.mark.parametrize("text", STAGED)
def test_mirrored_box_decomposition_matches_oracle(text):
    """h = source position -> destination position for (layout -> row-major):
    h(q*B + r) == base(q) + row(r)*SX + col(r) == the oracle's inverse map."""
    g = L.parse_layout(text)
    spec = O.parse(text)
    fh, h, n_src, n_dst = lower.gather_expr(None, g)
    bp = staging.box_plan(h, fh, n_src, n_dst, 4)
    q = np.arange(n_src, dtype=np.int64) // bp.block
    off = np.tile(bp.offsets.astype(np.int64), n_src // bp.block)
    got = staging.eval_vec(bp.base, {"q": q}) + (off // bp.pitch) * bp.sx + off % bp.pitch
    np.testing.assert_array_equal(got, O.inv_range(spec))


def test_f1_bench_layout_plans_staged():
    f1 = L.parse_layout("GroupBy([8192,8192]).OrderBy(RegP([128,64,128,64],[1,3,2,4]))"
                        ".OrderBy(RegP([128,128],[2,1]), GenP([64,64], antidiag))")
    for elem in (1, 2, 4, 8):
        p = K.plan_remap(None, f1, elem)
        assert p.kind == runtime.KIND_STAGED, p
        assert f"x64 (stride 8192" in p.detail


def test_contiguous_and_transposes_do_not_stage():
    row = L.parse_layout("GroupBy([64,64])")
    f, g, n, m = lower.gather_expr(None, row)
    assert staging.box_plan(g, f, n, m, 4) is None
    col = L.parse_layout("GroupBy([1024,1024]).OrderBy(Col(1024,1024))")
    assert K.plan_remap(None, col, 2).kind == runtime.KIND_TRANSPOSE


def test_eval_vec_matches_exact_evaluator():
    g = L.parse_layout(STAGED[0])
    f, gx, n_dst, _ = lower.gather_expr(None, g)
    rng = np.random.default_rng(3)
    xs = rng.integers(0, n_dst, 300)
    got = staging.eval_vec(gx, {"f": xs})
    want = [eval_expr(gx, {"f": int(x)}) for x in xs]
    assert got.tolist() == want
    # the anti-diagonal inverse (isqrt + selects) over its whole domain
    a = L.parse_layout("GroupBy([96,96]).OrderBy(GenP([96,96], antidiag))")
    f, inv = lower.inv_map_expr(a)
    allf = np.arange(96 * 96)
    assert staging.eval_vec(inv, {"f": allf}).tolist() == O.inv_range(O.parse(
        "GroupBy([96,96]).OrderBy(GenP([96,96], antidiag))")).tolist()


# ---------------------------------------------------------------------------
# GPU
# ---------------------------------------------------------------------------

NP = {1: np.int8, 2: np.int16, 4: np.int32, 8: np.int64}


def _torch():
    return pytest.importorskip("torch")


@pytest.mark.gpu
@pytest.mark.parametrize("text", STAGED)
@pytest.mark.parametrize("elem", [1, 2, 4, 8])
def test_staged_remap_vs_oracle(text, elem):
    torch = _torch()
    g = L.parse_layout(text)
    spec = O.parse(text)
    n = O.logical_size(spec)
    batch = 3
    host = (np.arange(batch * n, dtype=np.int64) * 2654435761 % (1 << 31)).astype(NP[elem])
    host = host.reshape(batch, n)
    got = K.remap(torch.from_numpy(host).cuda(), None, g).cpu().numpy()
    for b in range(batch):
        np.testing.assert_array_equal(got[b], O.remap(host[b], None, spec, dst_size=n))
    # layout -> row-major (mirrored: source blocks into destination boxes)
    back = K.remap(torch.from_numpy(host).cuda(), g, None).cpu().numpy()
    for b in range(batch):
        np.testing.assert_array_equal(back[b], O.remap(host[b], spec, None, dst_size=n))


@pytest.mark.gpu
@pytest.mark.parametrize("elem", [2, 4])
def test_staged_unaligned_source_takes_scalar_loads(elem):
    """A source that is element- but not 16-byte-aligned: the kernel's
    per-CTA alignment check routes the box loads to the scalar path."""
    torch = _torch()
    text = STAGED[2]
    g = L.parse_layout(text)
    spec = O.parse(text)
    n = O.logical_size(spec)
    host = (np.arange(n + 1, dtype=np.int64) * 7919 % 30011).astype(NP[elem])
    dev = torch.from_numpy(host).cuda()[1:]
    assert dev.data_ptr() % 16
    got = K.remap(dev, None, g).cpu().numpy()
    np.testing.assert_array_equal(got, O.remap(host[1:], None, spec, dst_size=n))
    # mirrored kernel: unaligned source and destination
    out = torch.zeros(n + 1, dtype=dev.dtype, device="cuda")[1:]
    K.remap(dev, g, None, out=out)
    np.testing.assert_array_equal(out.cpu().numpy(), O.remap(host[1:], spec, None, dst_size=n))


@pytest.mark.gpu
def test_staged_f1_full_size():
    """SURVEY f1 at the bench size (8192^2 int32): scatter into the layout is
    src[inv_map]; gathering back restores the source."""
    torch = _torch()
    f1 = L.parse_layout("GroupBy([8192,8192]).OrderBy(RegP([128,64,128,64],[1,3,2,4]))"
                        ".OrderBy(RegP([128,128],[2,1]), GenP([64,64], antidiag))")
    assert K.remap_plan(None, f1, 4).kind == runtime.KIND_STAGED
    n = 8192 * 8192
    src = torch.arange(n, dtype=torch.int32, device="cuda")
    fwd = K.remap(src, None, f1)
    inv = K.inv_map(f1, dtype=torch.int64)
    assert torch.equal(fwd, src[inv])
    back = K.remap(fwd, f1, None)
    assert torch.equal(back, src)
    # a window against the oracle
    spec = O.parse("GroupBy([8192,8192]).OrderBy(RegP([128,64,128,64],[1,3,2,4]))"
                   ".OrderBy(RegP([128,128],[2,1]), GenP([64,64], antidiag))")
    want = O.inv_range(spec, first=12345 * 4096, count=3 * 4096)
    np.testing.assert_array_equal(fwd[12345 * 4096:12348 * 4096].cpu().numpy(), want)


TWO = [
    ("GroupBy([256,256]).OrderBy(RegP([4,64,4,64],[1,3,2,4])).OrderBy(RegP([4,4],[2,1]), GenP([64,64], antidiag))",
     "GroupBy([256,256]).OrderBy(RegP([8,32,8,32],[1,3,2,4]))"),
    ("GroupBy([256,256]).OrderBy(RegP([4,64,4,64],[1,3,2,4])).OrderBy(RegP([4,4],[2,1]), GenP([64,64], antidiag))",
     "GroupBy([256,256]).OrderBy(Col(256,256))"),
]


@pytest.mark.parametrize("a,b", TWO)
def test_two_layout_remaps_plan_staged(a, b):
    la, lb = L.parse_layout(a), L.parse_layout(b)
    for s_, d_ in ((la, lb), (lb, la)):
        for elem in (2, 4):
            assert K.plan_remap(s_, d_, elem).kind == runtime.KIND_STAGED


@pytest.mark.gpu
@pytest.mark.parametrize("a,b", TWO)
@pytest.mark.parametrize("elem", [2, 4])
def test_two_layout_staged_remaps_vs_oracle(a, b, elem):
    torch = _torch()
    sa, sb = O.parse(a), O.parse(b)
    la, lb = L.parse_layout(a), L.parse_layout(b)
    n = O.size(sa)
    host = (np.arange(2 * n, dtype=np.int64) * 40503 % 65521).astype(NP[elem]).reshape(2, n)
    for (ls, ss), (ld, sd) in (((la, sa), (lb, sb)), ((lb, sb), (la, sa))):
        got = K.remap(torch.from_numpy(host).cuda(), ls, ld).cpu().numpy()
        for k in range(2):
            np.testing.assert_array_equal(got[k], O.remap(host[k], ss, sd, dst_size=n))


@pytest.mark.gpu
@pytest.mark.parametrize("elem", [1, 2, 4, 8])
def test_bulk_staged_variant_vs_oracle(elem, monkeypatch):
    """The TMA-fed persistent variant (cp.async.bulk box rows, off by
    default) stays bit-exact, aligned and unaligned sources."""
    torch = _torch()
    monkeypatch.setattr(staging, "BOX_BULK", 1)
    text = STAGED[2]
    g = L.parse_layout(text)
    spec = O.parse(text)
    n = O.logical_size(spec)
    assert "TMA bulk" in K.remap_plan(None, g, elem).detail
    host = (np.arange(n + 1, dtype=np.int64) * 2654435761 % 100003).astype(NP[elem])
    dev = torch.from_numpy(host).cuda()
    for view, h in ((dev[:n], host[:n]), (dev[1:], host[1:])):
        got = K.remap(view.contiguous() if view.data_ptr() % 16 == 0 else view, None, g).cpu().numpy()
        np.testing.assert_array_equal(got, O.remap(h, None, spec, dst_size=n))


@pytest.mark.gpu
def test_staged_beyond_int32_positions():
    """A staged layout with more than 2^31 positions (int8, 46400^2): 64-bit
    block origins; sampled positions against the scalar layout API, and the
    size-independent round trip through the mirrored kernel."""
    torch = _torch()
    text = ("GroupBy([46400,46400]).OrderBy(RegP([725,64,725,64],[1,3,2,4]))"
            ".OrderBy(RegP([725,725],[2,1]), GenP([64,64], antidiag))")
    g = L.parse_layout(text)
    assert K.remap_plan(None, g, 1).kind == runtime.KIND_STAGED
    n = 46400
    assert n * n > 2 ** 31
    x = torch.randint(-128, 128, (n * n,), dtype=torch.int8, device="cuda")
    y = K.remap(x, None, g)
    rng = np.random.default_rng(7)
    ij = rng.integers(0, n, size=(2000, 2))
    pos = torch.tensor([g.apply((int(i), int(j))) for i, j in ij], device="cuda")
    flat = torch.tensor([int(i) * n + int(j) for i, j in ij], device="cuda")
    assert torch.equal(y[pos], x[flat])
    back = K.remap(y, g, None)
    assert torch.equal(back, x)
    del x, y, back
    torch.cuda.empty_cache()
