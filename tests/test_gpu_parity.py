"""GPU parity: the CUDA path (through the C ABI) against the oracle and the
reference's own golden vectors.  Bit-exact for every index map and remap."""

import hashlib

import numpy as np
import pytest

from conftest import golden
from helpers_spec import layout_from_spec

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2505_08091_b200 as L  # noqa: E402
from paper_2505_08091_b200 import kernels as K  # noqa: E402
from oracle import oracle as O  # noqa: E402

SMALL = [n for n, c in golden().items() if "apply" in c]
ALL = list(golden())
BIG = [n for n, c in golden().items() if c["logical_size"] > 1 << 20]


def _layout(c):
    return L.parse_layout(c["dsl"]) if c.get("dsl") else layout_from_spec(c["spec"])


def _sha(t):
    h = hashlib.sha256()
    step = 1 << 24
    for lo in range(0, t.numel(), step):
        h.update(t[lo:lo + step].to(torch.int64).cpu().numpy().astype("<i8").tobytes())
    return h.hexdigest()


@pytest.mark.parametrize("name", SMALL)
def test_index_maps_full_tables(name):
    c = golden()[name]
    g = _layout(c)
    assert K.apply_map(g).cpu().tolist() == c["apply"]
    assert K.inv_map(g).cpu().tolist() == c["inv"]
    assert K.apply_map(g, dtype=torch.int64).cpu().tolist() == c["apply"]


@pytest.mark.parametrize("name", ALL)
def test_index_maps_against_reference_digest_and_samples(name):
    c = golden()[name]
    g = _layout(c)
    app = K.apply_map(g)
    inv = K.inv_map(g)
    s = c["samples"]
    assert app[torch.tensor(s["x"], device=app.device)].cpu().tolist() == s["apply"]
    assert inv[torch.tensor(s["f"], device=inv.device)].cpu().tolist() == s["inv"]
    if "apply_sha256" in c:
        assert _sha(app) == c["apply_sha256"]
        assert _sha(inv) == c["inv_sha256"]


@pytest.mark.parametrize("name", ALL)
def test_bijective_on_device(name):
    g = _layout(golden()[name])
    assert K.check_bijective(g)


def test_non_bijective_genp_detected():
    def fwd(idx):
        return (idx[0] * 2) % 64

    bad = L.GenP((64,), L.PermFn(fwd, lambda idx: (idx[0] * 2) % 64),
                 L.PermFn(lambda f: (f,), lambda f: (f,)), name="collide")
    g = L.GroupBy([64], orders=(L.OrderBy(bad),))
    assert not K.check_bijective(g)


def _check_remap(src_spec, dst_spec, src_layout, dst_layout, dtype, batch=1):
    some = src_spec or dst_spec
    n_src = O.size(src_spec) if src_spec else O.logical_size(some)
    n_dst = O.size(dst_spec) if dst_spec else O.logical_size(some)
    info = torch.iinfo(dtype)
    host = np.arange(batch * n_src, dtype=np.int64)
    if dtype != torch.int64:
        host = host % (info.max - info.min + 1) + info.min
    host = host.astype({torch.int8: np.int8, torch.int16: np.int16, torch.int32: np.int32,
                        torch.int64: np.int64}[dtype]).reshape(batch, n_src)
    src = torch.from_numpy(host).cuda()
    got = K.remap(src, src_layout, dst_layout).cpu().numpy()
    for b in range(batch):
        want = O.remap(host[b], src_spec, dst_spec, dst_size=n_dst)
        if dst_spec and dst_spec["kind"] == "expand":
            pass
        np.testing.assert_array_equal(got[b], want)


REMAP_CASES = [(n, dt) for k, n in enumerate(x for x in ALL if golden()[x]["logical_size"] <= 1 << 20)
               for dt in (("int16", "int32") if k % 4 else ("int8", "int16", "int32", "int64"))]


@pytest.mark.parametrize("name,dtype", REMAP_CASES)
def test_scatter_gather_vs_oracle(name, dtype):
    c = golden()[name]
    if c["spec"]["kind"] == "expand":
        pytest.skip("ExpandBy remaps are covered by test_expand_remap")
    dt = getattr(torch, dtype)
    g = _layout(c)                 # ragged sizes take the scalar gather / scatter kernels
    _check_remap(None, c["spec"], None, g, dt, batch=2)
    _check_remap(c["spec"], None, g, None, dt, batch=1)


def test_remap_between_two_layouts():
    a = "GroupBy([64,64]).OrderBy(RegP([2,32,2,32],[1,3,2,4]))"
    b = "GroupBy([64,64]).OrderBy(Col(64,64))"
    _check_remap(O.parse(a), O.parse(b), L.parse_layout(a), L.parse_layout(b), torch.int16, 3)
    _check_remap(O.parse(b), O.parse(a), L.parse_layout(b), L.parse_layout(a), torch.int32, 1)


def test_expand_remap():
    text = "ExpandBy([30,28],[32,32],GroupBy([32,32]).OrderBy(RegP([2,16,2,16],[1,3,2,4])))"
    g = L.parse_layout(text)
    spec = O.parse(text)
    # gather: physical (ExpandBy) buffer -> logical row-major; masked slots read as 0
    n_phys = O.size(spec)
    host = np.arange(n_phys, dtype=np.int32) + 1
    got = K.remap(torch.from_numpy(host).cuda(), g, None).cpu().numpy()
    want = O.remap(host, spec, None, dst_size=O.logical_size(spec))
    np.testing.assert_array_equal(got, want)


@pytest.mark.parametrize("name", BIG)
@pytest.mark.parametrize("dtype", ["int16", "int32"])
def test_bench_layout_remaps_full_size(name, dtype):
    """Full-size bench layouts, unique bit patterns, both directions, exact."""
    c = golden()[name]
    g = _layout(c)
    dt = getattr(torch, dtype)
    n = c["size"]
    src = torch.arange(n, dtype=torch.int64, device="cuda").to(dt)
    fwd = K.remap(src, None, g)                 # scatter into the layout
    back = K.remap(fwd, g, None)                # gather back to row-major
    assert torch.equal(back, src)
    # fwd[apply(x)] == src[x] <=> fwd == src[inv_map]
    inv = K.inv_map(g, dtype=torch.int64)
    assert torch.equal(fwd, src[inv])
    # and the oracle agrees on a window of the layout
    spec = c["spec"]
    host = src.cpu().numpy()
    want = O.remap(host, None, spec, dst_size=n)
    np.testing.assert_array_equal(fwd.cpu().numpy(), want)


def test_softmax_vs_float64():
    torch.manual_seed(2)
    for rows, cols in ((8192, 8192), (7, 4), (33, 1028), (3, 65536)):
        x = torch.randn(rows, cols, device="cuda") * 4
        y = K.softmax(x)
        want = O.softmax_rows_f64(x.cpu().numpy())
        rel = np.abs(y.cpu().numpy() - want) / np.maximum(want, 1e-30)
        assert rel.max() <= 1e-5, (rows, cols, rel.max())


def test_errors_map_to_reference_exceptions():
    g = L.parse_layout("GroupBy([64,64]).OrderBy(Col(64,64))")
    with pytest.raises(L.OutOfBounds):
        K.apply_map(g, first=4000, count=200)
    with pytest.raises(L.ShapeMismatch):
        K.remap(torch.zeros(100, device="cuda"), None, g)
    with pytest.raises(L.ArityMismatch):
        K.remap(torch.zeros(4096, device="cuda"), L.parse_layout("GroupBy([4096])"), g)


def test_injective_layout_scatter():
    """Injective-mode layouts (no inverse) scatter: dst[apply(x)] = src[x]
    (reference layout.py:304-311; test_layout.py even-map)."""
    def even(shape):
        return L.GenP(shape, L.PermFn(lambda idx: idx[0] * 2, lambda idx: idx[0] * 2), None, name="even")

    g = L.GroupBy([64], orders=(L.OrderBy(even((64,))),), injective=True)
    src = torch.arange(64, dtype=torch.int32, device="cuda") + 1
    out = K.remap(src, None, g).cpu().numpy()
    want = np.zeros(127, dtype=np.int32)
    want[0::2] = np.arange(64) + 1
    np.testing.assert_array_equal(out, want)
    assert K.apply_map(g).cpu().tolist() == [2 * i for i in range(64)]


def test_expand_scatter_and_roundtrip():
    text = "ExpandBy([30,28],[32,32],GroupBy([32,32]).OrderBy(RegP([2,16,2,16],[1,3,2,4])))"
    g = L.parse_layout(text)
    spec = O.parse(text)
    n_log = O.logical_size(spec)
    host = np.arange(n_log, dtype=np.int32) + 1
    got = K.remap(torch.from_numpy(host).cuda(), None, g).cpu().numpy()
    want = O.remap(host, None, spec, dst_size=O.size(spec))
    np.testing.assert_array_equal(got, want)


@pytest.mark.parametrize("dsl", [
    # multi-stage chains with in-tile GenPs, at a few hundred thousand points
    "GroupBy([512,512]).OrderBy(RegP([16,32,16,32],[1,3,2,4])).OrderBy(RegP([16,16],[2,1]), GenP([32,32], antidiag))",
    "GroupBy([384,256]).OrderBy(RegP([384,256],[2,1])).OrderBy(RegP([2,128,3,128],[3,1,4,2]))",
    "TileOrderBy(Col(16,16), Row(32,32))",
])
def test_multistage_chains_vs_oracle(dsl):
    g = L.parse_layout(dsl)
    spec = O.parse(dsl)
    assert np.array_equal(K.apply_map(g, dtype=torch.int64).cpu().numpy(), O.apply_range(spec))
    assert np.array_equal(K.inv_map(g, dtype=torch.int64).cpu().numpy(), O.inv_range(spec))
    _check_remap(None, spec, None, g, torch.int32, batch=2)
    _check_remap(spec, None, g, None, torch.int16, batch=1)
    assert K.check_bijective(g)


def test_remap_beyond_int32_positions():
    """A layout with more than 2^31 positions (64-bit index arithmetic in the
    generated maps): sampled positions against the closed form, and the
    size-independent round trip remap(remap(x, -> L), L ->) == x."""
    n = 46341                                   # n^2 = 2_147_488_281 > 2^31, odd: ragged path
    g = L.parse_layout(f"GroupBy([{n},{n}]).OrderBy(Col({n},{n}))")
    x = torch.randint(-128, 128, (n * n,), dtype=torch.int8, device="cuda")
    y = K.remap(x, None, g)
    idx = torch.randint(0, n, (2, 1 << 20), device="cuda")
    i, j = idx[0].long(), idx[1].long()
    assert torch.equal(y[j * n + i], x[i * n + j])
    back = K.remap(y, g, None)
    assert torch.equal(back, x)
    del x, y, back
    torch.cuda.empty_cache()
