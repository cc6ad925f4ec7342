"""A seeded corpus of 60 random layouts (tests/random_layouts.py): the Python
frontend against the C oracle on CPU, and the CUDA index maps and remaps
against the oracle on the GPU (bit-exact)."""

import numpy as np
import pytest

from oracle import oracle as O
from random_layouts import corpus

import paper_2505_08091_b200 as L

CORPUS = corpus()


@pytest.mark.parametrize("text", CORPUS[::3])
def test_frontend_matches_oracle(text):
    g = L.parse_layout(text)
    spec = O.parse(text)
    n = O.logical_size(spec)
    dims = O.dims(spec)
    pts = np.linspace(0, n - 1, num=min(n, 512), dtype=np.int64)
    app = O.apply_range(spec)
    inv = O.inv_range(spec)
    for x in pts:
        idx = tuple(int(v) for v in np.unravel_index(int(x), dims))
        assert g.apply(idx) == app[x]
        assert tuple(g.inv(int(x))) == tuple(int(v) for v in np.unravel_index(int(inv[x]), dims))


@pytest.mark.gpu
@pytest.mark.parametrize("text", CORPUS)
def test_device_maps_and_remaps_match_oracle(text):
    torch = pytest.importorskip("torch")
    from paper_2505_08091_b200 import kernels as K
    g = L.parse_layout(text)
    spec = O.parse(text)
    assert np.array_equal(K.apply_map(g).cpu().numpy(), O.apply_range(spec))
    assert np.array_equal(K.inv_map(g).cpu().numpy(), O.inv_range(spec))
    n = O.logical_size(spec)
    for dt, npdt in ((torch.int16, np.int16), (torch.int32, np.int32)):
        host = (np.arange(2 * n, dtype=np.int64) % 30011).astype(npdt).reshape(2, n)
        src = torch.from_numpy(host).cuda()
        fwd = K.remap(src, None, g).cpu().numpy()
        back = K.remap(src, g, None).cpu().numpy()
        for b in range(2):
            assert np.array_equal(fwd[b], O.remap(host[b], None, spec)), (text, dt)
            assert np.array_equal(back[b], O.remap(host[b], spec, None)), (text, dt)


EXPAND = __import__("random_layouts").expand_corpus()


@pytest.mark.parametrize("text", EXPAND[::3])
def test_frontend_expand_matches_oracle(text):
    g = L.parse_layout(text)
    spec = O.parse(text)
    dims = O.dims(spec)
    app = O.apply_range(spec)
    for x in range(O.logical_size(spec)):
        got = g.apply(tuple(int(v) for v in np.unravel_index(x, dims)))
        assert (-1 if got is None else got) == app[x]


@pytest.mark.gpu
@pytest.mark.parametrize("text", EXPAND)
def test_device_expand_maps_and_gather_match_oracle(text):
    torch = pytest.importorskip("torch")
    from paper_2505_08091_b200 import kernels as K
    g = L.parse_layout(text)
    spec = O.parse(text)
    assert np.array_equal(K.apply_map(g).cpu().numpy(), O.apply_range(spec))
    assert np.array_equal(K.inv_map(g).cpu().numpy(), O.inv_range(spec))
    # gather: physical (partial-tile) buffer -> logical row-major, masked slots read 0
    host = np.arange(O.size(spec), dtype=np.int32) + 1
    got = K.remap(torch.from_numpy(host).cuda(), g, None).cpu().numpy()
    assert np.array_equal(got, O.remap(host, spec, None, dst_size=O.logical_size(spec)))


CHAINS = __import__("random_layouts").chain_corpus()


@pytest.mark.parametrize("text", CHAINS[::4])
def test_frontend_chain_matches_oracle(text):
    g = L.parse_layout(text)
    spec = O.parse(text)
    n = O.logical_size(spec)
    dims = O.dims(spec)
    app = O.apply_range(spec)
    for x in np.linspace(0, n - 1, num=64, dtype=np.int64):
        idx = tuple(int(v) for v in np.unravel_index(int(x), dims))
        assert g.apply(idx) == app[x]


@pytest.mark.gpu
@pytest.mark.parametrize("text", CHAINS)
def test_device_chain_remaps_match_oracle(text):
    """Larger two-stage chains (up to 2^20 points): whichever kernel the
    planner picks (staged box, transpose, gather), both directions, int16 and
    int32, batch 2, bit-exact against the oracle."""
    torch = pytest.importorskip("torch")
    from paper_2505_08091_b200 import kernels as K
    g = L.parse_layout(text)
    spec = O.parse(text)
    n = O.logical_size(spec)
    for dt, npdt in ((torch.int32, np.int32), (torch.int16, np.int16)):
        host = (np.arange(2 * n, dtype=np.int64) * 2654435761 % 65521).astype(npdt).reshape(2, n)
        dev = torch.from_numpy(host).cuda()
        fwd = K.remap(dev, None, g).cpu().numpy()
        back = K.remap(dev, g, None).cpu().numpy()
        for b in range(2):
            np.testing.assert_array_equal(fwd[b], O.remap(host[b], None, spec, dst_size=n))
            np.testing.assert_array_equal(back[b], O.remap(host[b], spec, None, dst_size=n))
