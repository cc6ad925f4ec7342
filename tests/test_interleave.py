"""Register interleaves (lower.narrow_plan, LEGO_NARROW): digit permutations
whose innermost source or destination digit spans less than a 16-byte
vector -- AoS <-> SoA / AoSoA conversions -- regrouped in registers.

CPU: the planner's choice and the inverse map it builds; GPU: bit-exact
against the C oracle for 1- to 8-byte elements, both directions."""

import random

import numpy as np
import pytest

import paper_2505_08091_b200 as L
from paper_2505_08091_b200 import kernels as K, lower
from paper_2505_08091_b200.expr import eval_expr

LAYOUTS = [
    "GroupBy([8192,32,4]).OrderBy(RegP([8192,32,4],[1,3,2]))",        # AoS -> AoSoA, 4 channels
    "GroupBy([16384,32,2]).OrderBy(RegP([16384,32,2],[1,3,2]))",      # complex split in 32-groups
    "GroupBy([32768,8,4]).OrderBy(RegP([32768,8,4],[1,3,2]))",
    "GroupBy([512,512,4]).OrderBy(RegP([512,512,4],[3,1,2]))",        # RGBA planar <-> packed
]


@pytest.mark.parametrize("dsl", LAYOUTS)
def test_plans_and_inverse_maps(dsl):
    g = L.parse_layout(dsl)
    for e in (1, 2):
        for a, b in ((None, g), (g, None)):
            f, gg, nd, _ = lower.gather_expr(a, b)
            npl = lower.narrow_plan(gg, f, nd, e)
            if npl is None:
                continue
            assert 16 // npl.small >= 4
            if npl.mode == 1:                      # map = the inverse of the gather
                for fv in random.Random(0).sample(range(nd), 300):
                    assert eval_expr(npl.map, {"s": eval_expr(gg, {"f": fv})}) == fv
    assert "interleave" in repr(K.plan_remap(None, g, 1)) or "interleave" in repr(K.plan_remap(g, None, 1))


@pytest.mark.gpu
@pytest.mark.parametrize("dsl", LAYOUTS)
@pytest.mark.parametrize("dt", ["int8", "int16", "int32", "int64"])
def test_interleave_remaps_vs_oracle(dsl, dt):
    torch = pytest.importorskip("torch")
    from oracle import oracle as O
    g = L.parse_layout(dsl)
    spec = O.parse(dsl)
    n = O.logical_size(spec)
    host = (np.arange(n, dtype=np.int64) * 2654435761 % 1000003).astype(dt)
    x = torch.from_numpy(host).cuda()
    to = K.remap(x, None, g).cpu().numpy()
    assert np.array_equal(to, O.remap(host, None, spec))
    back = K.remap(torch.from_numpy(to).cuda(), g, None).cpu().numpy()
    assert np.array_equal(back, host)
