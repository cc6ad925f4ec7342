"""Pin the CPU oracle against vectors produced by the reference itself
(tests/golden/make_golden.py).  An oracle that disagrees with these is not
allowed to judge the CUDA path."""

import hashlib

import numpy as np
import pytest

from conftest import golden
from oracle import oracle as O

SMALL = [n for n, c in golden().items() if "apply" in c]
SAMPLED = [n for n, c in golden().items() if "samples" in c]


def _sha(chunks):
    h = hashlib.sha256()
    for c in chunks:
        h.update(np.ascontiguousarray(c, dtype="<i8").tobytes())
    return h.hexdigest()


@pytest.mark.parametrize("name", SMALL)
def test_full_tables(name):
    c = golden()[name]
    assert list(O.apply_range(c["spec"])) == c["apply"]
    assert list(O.inv_range(c["spec"])) == c["inv"]


@pytest.mark.parametrize("name", SAMPLED)
def test_sampled_points(name):
    c = golden()[name]
    s = c["samples"]
    app = O.apply_range(c["spec"])[s["x"]] if c["logical_size"] <= 1 << 22 else np.array(
        [O.apply_range(c["spec"], x, 1)[0] for x in s["x"]])
    assert list(app) == s["apply"]
    inv = np.array([O.inv_range(c["spec"], f, 1)[0] for f in s["f"]])
    assert list(inv) == s["inv"]


@pytest.mark.parametrize("name", [n for n, c in golden().items()
                                  if "apply_sha256" in c and c["logical_size"] <= 1 << 24])
def test_digests(name):
    c = golden()[name]
    step = 1 << 22
    n, m = c["logical_size"], c["size"]
    assert _sha(O.apply_range(c["spec"], lo, min(step, n - lo)) for lo in range(0, n, step)) \
        == c["apply_sha256"]
    assert _sha(O.inv_range(c["spec"], lo, min(step, m - lo)) for lo in range(0, m, step)) \
        == c["inv_sha256"]


@pytest.mark.slow
@pytest.mark.parametrize("name", [n for n, c in golden().items()
                                  if "apply_sha256" in c and c["logical_size"] > 1 << 24])
def test_digests_full_size(name):
    """2^28-point bench layouts, exhaustively (about 10-20 s each)."""
    test_digests(name)


def test_dsl_parser_matches_reference_specs():
    for name, c in golden().items():
        if c.get("dsl"):
            assert O.parse(c["dsl"]) == c["spec"], name


def test_reference_anchor_values():
    # test_acceptance.py:56-63, test_layout.py:36-39
    s = O.parse("GroupBy([6,4]).OrderBy(RegP([2,2],[2,1]), GenP([3,2], rev2d))")
    assert O.py_apply(s, (4, 1)) == 6
    assert O.apply_range(s)[4 * 4 + 1] == 6
    s = O.parse("GroupBy([6,6]).OrderBy(RegP([2,3,2,3],[1,3,2,4]))"
                ".OrderBy(RegP([2,2],[2,1]), GenP([3,3], antidiag))")
    assert O.apply_range(s)[4 * 6 + 2] == 15
    assert O.inv_range(s)[15] == 4 * 6 + 2


def test_python_and_c_restatements_agree():
    for name, c in golden().items():
        if c["logical_size"] > 5000:
            continue
        dims = c["dims"]
        from helpers_spec import unflat
        want = O.apply_range(c["spec"])
        got = [O.py_apply(c["spec"], unflat(dims, x)) for x in range(c["logical_size"])]
        assert [(-1 if g is None else g) for g in got] == list(want), name


def test_nw_sweep_matches_rowmajor():
    rng = np.random.default_rng(4)
    sim = rng.integers(-10, 11, size=(257, 257), dtype=np.int32)
    assert np.array_equal(O.nw(sim, 10), O.nw(sim, 10, rowmajor=True))


def test_remap_matches_table():
    c = golden()["cfg1_small"]
    src = np.arange(c["logical_size"], dtype=np.int32)
    dst = O.remap(src, None, c["spec"])
    want = np.empty_like(src)
    want[np.asarray(c["apply"])] = src
    assert np.array_equal(dst, want)
