"""Scatters into injective-mode layouts (reference layout.py:304-311).

Three semantics for positions no logical index hits: kept (``out`` given,
``fill=None``: the merge scatter), or set to ``fill`` by the same launch --
one fused kernel writing whole 16-byte windows when the planner proves the
map affine (``apply(x) = k*x + c``), a vector fill pass + scatter otherwise.
All checked bit-exact against the concrete-callable oracle.
"""

import numpy as np
import pytest

import paper_2505_08091_b200 as L
from oracle import concrete as C


def _inj(n, f, fs=None):
    g = L.GenP((n,), L.PermFn(lambda i: f(i[0]), lambda i: (fs or f)(i[0])), None)
    return L.GroupBy([n], orders=(L.OrderBy(g),), injective=True)


def test_planner_proves_affine_maps():
    from paper_2505_08091_b200 import kernels as K
    assert "affine 2x+0" in K.plan_remap(None, _inj(1 << 12, lambda x: 2 * x), 4, fill=True).detail
    assert "affine 3x+4" in K.plan_remap(None, _inj(1 << 12, lambda x: 3 * x + 4), 4, fill=True).detail
    assert "fill pass" in K.plan_remap(None, _inj(1000, lambda x: x * x), 4, fill=True).detail
    # an offset that breaks 16-byte windows falls back to the fill pass
    assert "fill pass" in K.plan_remap(None, _inj(1 << 12, lambda x: 2 * x + 1), 4, fill=True).detail


CASES = [("even", 1 << 20, lambda x: 2 * x), ("stride3+4", 1 << 18, lambda x: 3 * x + 4),
         ("stride4", 4099 * 4, lambda x: 4 * x), ("square", 3000, lambda x: x * x),
         ("odd", 1 << 16, lambda x: 2 * x + 1)]


@pytest.mark.gpu
@pytest.mark.parametrize("name,n,f", CASES)
@pytest.mark.parametrize("dt", ["int8", "int16", "int32", "int64"])
def test_fill_modes(name, n, f, dt):
    torch = pytest.importorskip("torch")
    from paper_2505_08091_b200 import kernels as K
    lay = _inj(n, f)
    rng = np.random.default_rng(n)
    info = np.iinfo(dt)
    x = rng.integers(info.min, info.max, size=n, dtype=dt, endpoint=True)
    xd = torch.from_numpy(x).cuda()
    want0 = C.remap(x, None, lay)
    got = K.remap(xd, None, lay)                                       # fresh output: fill 0
    assert np.array_equal(got.cpu().numpy(), want0)
    hit = np.zeros(len(want0), bool)
    hit[C.apply_all(lay)] = True
    out = torch.full((len(want0),), 5, dtype=getattr(torch, dt), device="cuda")
    K.remap(xd, None, lay, out=out, fill=-3)                           # explicit fill
    want = np.where(hit, want0, np.array(-3, dtype=dt))
    assert np.array_equal(out.cpu().numpy(), want)
    out.fill_(5)
    K.remap(xd, None, lay, out=out)                                    # merge: unhit keep 5
    want = np.where(hit, want0, np.array(5, dtype=dt))
    assert np.array_equal(out.cpu().numpy(), want)
