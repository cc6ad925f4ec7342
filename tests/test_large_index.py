"""Index spaces past 2^31 points (maximum sizes): the reference computes with
Python integers (pkg/src/lego/expr.py:261-316), so positions of a 65536 x
65536 layout (2^32 points) must stay exact on the device.  The generated maps
switch to 64-bit arithmetic from the interval analysis; these tests pin the
top of the range against the C oracle and check a full 2^32-element remap
by its transpose and round trip."""
import numpy as np
import pytest
import torch

import paper_2505_08091_b200 as L
from oracle import oracle as O
from paper_2505_08091_b200 import kernels as K

pytestmark = pytest.mark.gpu

N = 65536
TAIL = 1 << 20


def _layouts():
    return {
        "col": f"GroupBy([{N},{N}]).OrderBy(Col({N},{N}))",
        "antidiag": f"GroupBy([{N},{N}]).OrderBy(GenP([{N},{N}], antidiag))",
        "tiled": f"GroupBy([{N},{N}]).OrderBy(RegP([{N // 64},64,{N // 64},64],[1,3,2,4]))",
    }


@pytest.mark.parametrize("name", ["col", "antidiag", "tiled"])
def test_index_maps_top_of_2p32(name):
    dsl = _layouts()[name]
    g = L.parse_layout(dsl)
    spec = O.parse(dsl)
    assert O.size(spec) == N * N
    for first in (0, (1 << 31) - TAIL // 2, N * N - TAIL):
        got = K.apply_map(g, dtype=torch.int64, first=first, count=TAIL).cpu().numpy()
        assert np.array_equal(got, O.apply_range(spec, first, TAIL)), (name, first)
        got = K.inv_map(g, dtype=torch.int64, first=first, count=TAIL).cpu().numpy()
        assert np.array_equal(got, O.inv_range(spec, first, TAIL)), (name, first)


def test_remap_2p32_int8_transpose_round_trip():
    g = L.parse_layout(_layouts()["col"])
    gen = torch.Generator(device="cuda").manual_seed(7)
    src = torch.randint(-128, 128, (N * N,), dtype=torch.int8, device="cuda", generator=gen)
    out = K.remap(src, None, g)
    assert torch.equal(out.view(N, N), src.view(N, N).t().contiguous())
    # positions from the oracle at the top of the range
    pos = O.apply_range(O.parse(_layouts()["col"]), N * N - TAIL, TAIL)
    idx = torch.from_numpy(pos).cuda()
    assert torch.equal(out[idx], src[N * N - TAIL:])
    del out
    back = K.remap(K.remap(src, None, g), g, None)
    assert torch.equal(back, src)
