"""Parity of arbitrary user-defined bijections at scale.

The reference semantics of a user GenP is its concrete callable
(layout.py:187-200).  oracle/concrete.py evaluates the reference algorithm
over whole index spaces with those callables; it is pinned here against
digests of full tables the REFERENCE ITSELF produced for the same layouts
(tests/golden/make_user_golden.py -> tests/golden/user_genps.json) and
against the reference-generated tables of tests/golden/layouts.json.

GPU: index maps and remaps (gather from and scatter into the layout, int8 to
int64 elements) of six user layouts of 2^20 points -- XOR swizzle, bit
reversal, Morton order, rectangular skewed diagonal, a tiled chain with an
in-tile XOR GenP, and the injective even map (scatter-only, the f4 row) --
bit-exact against that oracle.
"""

import hashlib
import json
import os

import numpy as np
import pytest

import paper_2505_08091_b200 as L
from conftest import golden
from oracle import concrete as C
from user_genps import FACTORIES

HERE = os.path.dirname(os.path.abspath(__file__))
with open(os.path.join(HERE, "golden", "user_genps.json")) as fh:
    GOLD = {c["name"]: c for c in json.load(fh)["cases"]}


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<i8").tobytes()).hexdigest()


@pytest.mark.parametrize("name", list(FACTORIES))
def test_concrete_oracle_matches_reference_tables(name):
    lay = FACTORIES[name](L)
    g = GOLD[name]
    app = C.apply_all(lay)
    s = g["samples"]
    assert app[s["x"]].tolist() == s["apply"]
    assert _sha(app) == g["apply_sha256"]
    if not g["injective"]:
        inv = C.inv_all(lay)
        assert inv[s["x"]].tolist() == s["inv"]
        assert _sha(inv) == g["inv_sha256"]


def _perm_from_spec(p):
    shape = p["shape"]
    if p["kind"] == "regp":
        return L.RegP(shape, p["sigma"])
    if p["kind"] == "identity":
        return L.identity_perm(shape)
    if p["kind"] == "rev":
        return L.reverse_perm(shape)
    return L.antidiag_perm(shape[0])


def _layout_from_spec(spec):
    if spec["kind"] == "expand":
        return L.ExpandBy(spec["physical"], spec["expanded"], _layout_from_spec(spec["inner"]))
    return L.GroupBy(*spec["tiles"], orders=tuple(L.OrderBy(*[_perm_from_spec(p) for p in st])
                                                  for st in spec["stages"]))


@pytest.mark.parametrize("name", [n for n, c in golden().items() if "apply" in c])
def test_concrete_oracle_matches_builtin_golden_tables(name):
    c = golden()[name]
    lay = _layout_from_spec(c["spec"])
    assert C.apply_all(lay).tolist() == [-1 if v is None else v for v in c["apply"]]
    assert C.inv_all(lay).tolist() == c["inv"]


@pytest.mark.parametrize("name", list(FACTORIES))
def test_symbolic_builders_agree_with_callables(name):
    """What the device runs (the symbolic builder, generated) agrees with the
    reference semantics (the callable) on a sample -- the check validate()
    skips above 4096 points."""
    lay = FACTORIES[name](L)
    x = L.Var("x", L.VarRange(0, L.GroupBy(*lay.tiles).size))
    from paper_2505_08091_b200 import lower
    e = lower.simplify(L.as_expr(lower.apply_flat(lay, x)))
    app = C.apply_all(lay)
    for v in np.linspace(0, len(app) - 1, 300).astype(int):
        assert L.eval_expr(e, {"x": int(v)}) == app[v]


DTYPES = ["int8", "int16", "int32", "int64"]


@pytest.mark.gpu
@pytest.mark.parametrize("name", list(FACTORIES))
def test_device_maps_and_remaps(name):
    torch = pytest.importorskip("torch")
    from paper_2505_08091_b200 import kernels as K
    lay = FACTORIES[name](L)
    app = C.apply_all(lay)
    assert np.array_equal(K.apply_map(lay, dtype=torch.int64).cpu().numpy(), app)
    inv = None if lay.injective else C.inv_all(lay)
    if lay.injective:
        with pytest.raises(L.LegoError):
            K.inv_map(lay)
    else:
        assert np.array_equal(K.inv_map(lay, dtype=torch.int64).cpu().numpy(), inv)
    n = len(app)
    rng = np.random.default_rng(3)
    for dt in DTYPES:
        info = np.iinfo(dt)
        x = rng.integers(info.min, info.max, size=n, dtype=dt, endpoint=True)
        xd = torch.from_numpy(x).cuda()
        got = K.remap(xd, None, lay).cpu().numpy()                   # scatter: out[apply(x)] = x
        want = np.zeros(got.size, dtype=dt)
        want[app] = x
        assert np.array_equal(got, want), (name, dt, "scatter")
        if not lay.injective:
            got = K.remap(xd, lay, None).cpu().numpy()               # gather: out[x] = src[apply(x)]
            assert np.array_equal(got, x[app]), (name, dt, "gather")
            assert np.array_equal(x[app][inv], x)


def test_disagreeing_symbolic_builder_is_rejected_before_any_program():
    """A user GenP above the reference's 4096-point trust bound whose symbolic
    builder (what the device runs) disagrees with its concrete callable (the
    reference semantics) is refused when a program is planned from it."""
    import paper_2505_08091_b200 as L
    from paper_2505_08091_b200 import GenP, PermFn, kernels as K

    def fwd(idx):
        i, j = idx
        return i * 128 + (j ^ 1)             # concrete: swap neighbouring columns

    def fwd_sym(idx):
        i, j = idx
        return i * 128 + j                   # symbolic: identity (wrong)

    def inv(f):
        return f // 128, (f % 128) ^ 1

    def inv_sym(f):
        return f // 128, f % 128

    bad = GenP((128, 128), PermFn(fwd, fwd_sym), PermFn(inv, inv_sym), name=None)
    g = L.GroupBy([128, 128]).order_by(bad)
    with pytest.raises(L.LegoError, match="symbolic"):
        K.plan_remap(None, g, 4)
    with pytest.raises(L.LegoError, match="symbolic"):
        K.index_map_source(g)
