"""Host-side mirror of the reference API: scalar apply/inv and the symbolic
path agree with the reference's own outputs (golden vectors)."""

import random

import pytest

import paper_2505_08091_b200 as L
from conftest import golden
from helpers_spec import flat, layout_from_spec, unflat

SMALL = [n for n, c in golden().items() if "apply" in c]


def _layout(c):
    return L.parse_layout(c["dsl"]) if c.get("dsl") else layout_from_spec(c["spec"])


@pytest.mark.parametrize("name", SMALL)
def test_scalar_apply_inv_full_table(name):
    c = golden()[name]
    g = _layout(c)
    got = [g.apply(unflat(c["dims"], x)) for x in range(c["logical_size"])]
    assert [(-1 if v is None else v) for v in got] == c["apply"]
    assert [flat(c["dims"], g.inv(f)) for f in range(c["size"])] == c["inv"]


@pytest.mark.parametrize("name", [n for n, c in golden().items() if "apply" not in c])
def test_scalar_apply_inv_samples(name):
    c = golden()[name]
    g = _layout(c)
    s = c["samples"]
    assert [g.apply(unflat(c["dims"], x)) for x in s["x"]] == s["apply"]
    assert [flat(c["dims"], g.inv(f)) for f in s["f"]] == s["inv"]


@pytest.mark.parametrize("name", list(golden()))
def test_symbolic_matches_reference(name):
    c = golden()[name]
    g = _layout(c)
    names = [f"v{k}" for k in range(len(c["dims"]))]
    e = L.apply_symbolic(g, L.index_vars(names, c["dims"]))
    f = L.Var("f", L.VarRange(0, c["size"]))
    inv = L.inv_symbolic(g, f)
    s = c["samples"]
    for x, want in list(zip(s["x"], s["apply"]))[:200]:
        assert L.eval_expr(e, dict(zip(names, unflat(c["dims"], x)))) == want
    for fv, want in list(zip(s["f"], s["inv"]))[:200]:
        assert flat(c["dims"], [L.eval_expr(k, {"f": fv}) for k in inv]) == want


def test_reference_anchors_and_errors():
    g = L.parse_layout("GroupBy([6,4]).OrderBy(RegP([2,2],[2,1]), GenP([3,2], rev2d))")
    assert g.apply((4, 1)) == 6 and g.inv(6) == (4, 1)
    with pytest.raises(L.OutOfBounds):
        g.apply((6, 0))
    with pytest.raises(L.OutOfBounds):
        g.inv(24)
    with pytest.raises(L.ArityMismatch):
        g.apply((1, 2, 3))
    with pytest.raises(L.ShapeMismatch):
        L.parse_layout("GroupBy([4]).OrderBy(Row([5]))")
    with pytest.raises(L.UnknownBuiltinPerm):
        L.parse_layout("GroupBy([4]).OrderBy(GenP([4], nosuchperm))")
    with pytest.raises(L.LayoutSyntaxError) as err:
        L.parse_layout("GroupBy([6,4]).OrderBy(RegP([2,2],[2,1])")
    assert err.value.pos is not None
    x = L.parse_layout("ExpandBy([3,3],[4,4],GroupBy([4,4]).OrderBy(Col(4,4)))")
    assert x.apply((1, 2)) == 7 and x.apply((3, 3)) is None


def test_simplifier_sound_on_random_expressions():
    rng = random.Random(7)
    ops = ["add", "sub", "mul", "div", "mod", "sel"]

    def rand(vs, d):
        if d == 0 or rng.random() < 0.3:
            return rng.choice(vs) if rng.random() < 0.7 else L.IntConst(rng.randint(0, 9))
        k = rng.choice(ops)
        a = rand(vs, d - 1)
        if k == "add":
            return a + rand(vs, d - 1)
        if k == "sub":
            return a - rand(vs, d - 1)
        if k == "mul":
            return a * rand(vs, d - 1)
        if k == "div":
            return L.FloorDiv(a, rng.randint(1, 8))
        if k == "mod":
            return L.Mod(a, rng.randint(1, 8))
        return L.Select(L.lt(rand(vs, d - 1), rand(vs, d - 1)), a, rand(vs, d - 1))

    for _ in range(300):
        vs = [L.Var(f"v{k}", L.VarRange(rng.randint(-3, 0), rng.randint(2, 9)))
              for k in range(rng.randint(1, 2))]
        e = rand(vs, 4)
        s = L.simplify(e)
        import itertools
        for vals in itertools.product(*(range(v.range.lo, v.range.hi) for v in vs)):
            env = {v.name: x for v, x in zip(vs, vals)}
            assert L.eval_expr(s, env) == L.eval_expr(e, env), (e, s, env)
