"""Generate the golden vectors that pin the oracle -- run HERE, not on the GPU box.

Imports the *reference* package from ``/root/reference/pkg/src`` (read-only,
PUBLIC reference code; it is only executed, never copied) and records what its
own ``GroupBy.apply`` / ``inv`` (``layout.py:313-328``) and ``ExpandBy``
(``layout.py:383-400``) return:

* small layouts (the reference tests' anchors, the Table-I stride layouts,
  ExpandBy cases and the reference test-suite's random corpus
  ``helpers.layout_corpus(seed=20240901, count=30)``): full apply / inv
  tables when the layout has <= 4096 elements, otherwise 512 sampled points
  plus the SHA-256 of the full tables;
* the bench layouts at full size (BASELINE.json configs 1, 2, 4 and the NW
  block layout): 4096 sampled points evaluated with the reference's own
  per-element ``apply``/``inv``, plus full-table SHA-256 digests.  Config 1
  (2^24 points) is enumerated exhaustively with the reference ``apply`` on all
  cores; configs 2 and 4 (2^28 points) are enumerated by evaluating the
  reference's own emitted expression (``apply_symbolic`` -> ``emit_expr``
  with the triton profile, ``tl.where`` -> ``np.where``, exact ``isqrt``) in
  numpy, after checking that expression against the sampled ``apply``.

Output: ``tests/golden/layouts.json``.  Usage::

    python tests/golden/make_golden.py            # everything (~2-4 min)
    python tests/golden/make_golden.py --quick    # skip the 2^28 digests
"""

from __future__ import annotations

import argparse
import hashlib
import json
import math
import multiprocessing as mp
import os
import random
import sys
import time
from itertools import product

import numpy as np

REF_SRC = "/root/reference/pkg/src"
REF_TESTS = "/root/reference/pkg/tests"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "layouts.json")

sys.path.insert(0, REF_SRC)
sys.path.insert(0, REF_TESTS)

import lego  # noqa: E402  (the reference)
from lego.layout import ExpandBy, GenP, GroupBy, RegP  # noqa: E402

SMALL_FULL = 4096
N_SAMPLES_SMALL = 512
N_SAMPLES_BIG = 4096


def to_spec(layout):
    """Reference layout object -> oracle spec dict."""
    if isinstance(layout, ExpandBy):
        return {"kind": "expand", "physical": list(layout.physical),
                "expanded": list(layout.expanded), "inner": to_spec(layout.inner)}
    stages = []
    for o in layout.orders:
        stage = []
        for p in o.perms:
            if isinstance(p, RegP):
                stage.append({"kind": "regp", "shape": list(p.shape), "sigma": list(p.sigma)})
            elif isinstance(p, GenP):
                kind = {"identity": "identity", "rev": "rev", "antidiag": "antidiag"}[p.name]
                stage.append({"kind": kind, "shape": list(p.shape)})
            else:
                raise TypeError(p)
        stages.append(stage)
    return {"kind": "group", "tiles": [list(t) for t in layout.tiles], "stages": stages}


def unflat(shape, f):
    out = []
    for n in reversed(shape[1:]):
        out.append(f % n)
        f //= n
    out.append(f)
    return tuple(out[::-1])


def flat(shape, idx):
    acc = 0
    for c, n in zip(idx, shape):
        acc = acc * n + c
    return acc


def apply_flat(layout, x):
    r = layout.apply(unflat(layout.dims, x))
    return -1 if r is None else r


def inv_flat(layout, f):
    return flat(layout.dims, layout.inv(f))


def sha_of(chunks):
    h = hashlib.sha256()
    for c in chunks:
        h.update(np.ascontiguousarray(c, dtype="<i8").tobytes())
    return h.hexdigest()


def sample_points(n_logical, n_phys, k, rng, dims):
    """Random points plus the first/last rows and columns of the logical view."""
    xs = {0, n_logical - 1}
    if len(dims) >= 2:
        inner = dims[-1]
        for c in range(0, inner, max(1, inner // 64)):
            xs.add(c)
            xs.add(n_logical - inner + c)
        rows = n_logical // inner
        for r in range(0, rows, max(1, rows // 64)):
            xs.add(r * inner)
            xs.add(r * inner + inner - 1)
    while len(xs) < k:
        xs.add(rng.randrange(n_logical))
    fs = {0, n_phys - 1}
    while len(fs) < k:
        fs.add(rng.randrange(n_phys))
    return sorted(xs)[:max(k, len(xs))], sorted(fs)


def small_case(name, layout, dsl=None, rng=None):
    rng = rng or random.Random(hash(name) & 0xFFFF)
    n_log = math.prod(layout.dims)
    n_phys = layout.size
    case = {"name": name, "dsl": dsl, "spec": to_spec(layout), "dims": list(layout.dims),
            "size": n_phys, "logical_size": n_log}
    app = [apply_flat(layout, x) for x in range(n_log)]
    inv = [inv_flat(layout, f) for f in range(n_phys)]
    if n_log <= SMALL_FULL:
        case["apply"] = app
        case["inv"] = inv
    xs = sorted(rng.sample(range(n_log), min(N_SAMPLES_SMALL, n_log)))
    fs = sorted(rng.sample(range(n_phys), min(N_SAMPLES_SMALL, n_phys)))
    case["samples"] = {"x": xs, "apply": [app[x] for x in xs], "f": fs, "inv": [inv[f] for f in fs]}
    case["apply_sha256"] = sha_of([np.asarray(app)])
    case["inv_sha256"] = sha_of([np.asarray(inv)])
    return case


# --- exhaustive reference apply on all cores (config 1) ---------------------

_G = None


def _init(dsl):
    global _G
    _G = lego.parse_layout(dsl)


def _apply_chunk(bounds):
    lo, hi = bounds
    return np.fromiter((apply_flat(_G, x) for x in range(lo, hi)), dtype=np.int64, count=hi - lo)


def _inv_chunk(bounds):
    lo, hi = bounds
    return np.fromiter((inv_flat(_G, f) for f in range(lo, hi)), dtype=np.int64, count=hi - lo)


def exhaustive_reference(dsl, n, which):
    step = 1 << 18
    bounds = [(lo, min(n, lo + step)) for lo in range(0, n, step)]
    with mp.Pool(os.cpu_count(), initializer=_init, initargs=(dsl,)) as pool:
        fn = _apply_chunk if which == "apply" else _inv_chunk
        return sha_of(pool.imap(fn, bounds))


# --- numpy evaluation of the reference's emitted expression -----------------

def np_isqrt(x):
    r = np.floor(np.sqrt(x.astype(np.float64))).astype(np.int64)
    r = np.where(r * r > x, r - 1, r)
    r = np.where((r + 1) * (r + 1) <= x, r + 1, r)
    return r


class _TL:
    @staticmethod
    def where(c, a, b):
        return np.where(c, a, b)


def emitted_apply_fn(layout):
    names = [f"v{k}" for k in range(len(layout.dims))]
    e = lego.apply_symbolic(layout, lego.index_vars(names, layout.dims))
    text = lego.emit_expr(e, lego.TRITON_PROFILE)
    code = compile(text, "<emitted>", "eval")

    def fn(xs):
        env = dict(zip(names, unflat(layout.dims, xs)))
        env.update(tl=_TL, isqrt=np_isqrt)
        return np.asarray(eval(code, {}, env), dtype=np.int64) + np.zeros_like(xs)
    return fn, text


def emitted_inv_fn(layout):
    f = lego.Var("f", lego.VarRange(0, layout.size))
    coords = lego.inv_symbolic(layout, f)
    texts = [lego.emit_expr(c, lego.TRITON_PROFILE) for c in coords]
    codes = [compile(t, "<emitted>", "eval") for t in texts]

    def fn(fs):
        env = {"f": fs, "tl": _TL, "isqrt": np_isqrt}
        cs = [np.asarray(eval(c, {}, env), dtype=np.int64) + np.zeros_like(fs) for c in codes]
        return flat(layout.dims, cs)
    return fn, texts


def big_case(name, dsl, full, rng):
    t0 = time.time()
    layout = lego.parse_layout(dsl)
    n = layout.size
    case = {"name": name, "dsl": dsl, "spec": to_spec(layout), "dims": list(layout.dims),
            "size": n, "logical_size": n}
    xs, fs = sample_points(n, n, N_SAMPLES_BIG, rng, layout.dims)
    app = [apply_flat(layout, x) for x in xs]
    inv = [inv_flat(layout, f) for f in fs]
    case["samples"] = {"x": xs, "apply": app, "f": fs, "inv": inv}
    if full == "reference":
        case["apply_sha256"] = exhaustive_reference(dsl, n, "apply")
        case["inv_sha256"] = exhaustive_reference(dsl, n, "inv")
        case["digest_source"] = "reference GroupBy.apply/inv, exhaustive"
    elif full == "emitted":
        afn, atext = emitted_apply_fn(layout)
        ifn, itexts = emitted_inv_fn(layout)
        # the emitted expressions must reproduce the sampled reference values
        assert list(afn(np.asarray(xs, dtype=np.int64))) == app, name
        assert list(ifn(np.asarray(fs, dtype=np.int64))) == inv, name
        step = 1 << 24
        case["apply_sha256"] = sha_of(afn(np.arange(lo, min(n, lo + step), dtype=np.int64))
                                      for lo in range(0, n, step))
        case["inv_sha256"] = sha_of(ifn(np.arange(lo, min(n, lo + step), dtype=np.int64))
                                    for lo in range(0, n, step))
        case["digest_source"] = ("reference apply_symbolic/inv_symbolic emitted (triton profile) "
                                 "and evaluated exhaustively in numpy; checked against sampled "
                                 "reference apply/inv")
        case["emitted"] = {"apply": atext, "inv": itexts}
    print(f"  {name}: {time.time() - t0:.1f}s", flush=True)
    return case


SMALL_DSL = {
    # reference anchors (test_acceptance.py:43-63, test_layout.py:202-237)
    "tile_reverse": "GroupBy([6,4]).OrderBy(RegP([2,2],[2,1]), GenP([3,2], rev2d))",
    "antidiag_chain": ("GroupBy([6,6]).OrderBy(RegP([2,3,2,3],[1,3,2,4]))"
                       ".OrderBy(RegP([2,2],[2,1]), GenP([3,3], antidiag))"),
    # Table-I stride equivalences (test_acceptance.py:167-208)
    "tiling_6x6": "GroupBy([6,6]).OrderBy(RegP([2,3,2,3],[1,3,2,4]))",
    "bits5": "GroupBy([2,2,2,2,2]).OrderBy(RegP([2,2,2,2,2],[5,2,4,3,1]))",
    "coarsen": "GroupBy([2,2],[2,2]).OrderBy(Row(4,4))",
    "bricks": "GroupBy([4,4,4],[2,2,2]).OrderBy(Row(4,4,4), Row(2,2,2))",
    "tileby_8x8": "TileBy([2,2],[4,4]).OrderBy(Row(8,8))",
    "tile_order_by": "TileOrderBy(Col(2,2), Row(3,3))",
    "col_4x3": "GroupBy([4,3]).OrderBy(Col(3,4))",
    "matmul_blk": "GroupBy([2,2]).OrderBy(Col(2,2))",
    "matmul_axis": "TileBy([2],[4]).OrderBy(Row(8))",
    # ExpandBy (test_expandby.py, test_acceptance.py:270-293)
    "expand_col": "ExpandBy([3,3],[4,4],GroupBy([4,4]).OrderBy(Col(4,4)))",
    "expand_1d": "ExpandBy([3],[4],GroupBy([4]))",
    "expand_tile": "ExpandBy([5,7],[8,8],GroupBy([8,8]).OrderBy(RegP([2,4,2,4],[1,3,2,4])))",
    # antidiag sizes the reference pins (test_antidiag.py)
    **{f"antidiag_{n}": f"GroupBy([{n},{n}]).OrderBy(GenP([{n},{n}], antidiag))" for n in
       (1, 2, 3, 5, 8, 13, 16, 64)},
    # reduced-size versions of the bench layouts
    "cfg1_small": "GroupBy([64,64]).OrderBy(RegP([2,32,2,32],[1,3,2,4]))",
    "cfg2_small": "GroupBy([64,64]).OrderBy(Col(64,64))",
    "cfg2_rect": "GroupBy([48,80]).OrderBy(Col(80,48))",
    "nw_blocks_small": ("GroupBy([64,64]).OrderBy(RegP([4,16,4,16],[1,3,2,4]))"
                        ".OrderBy(GenP([4,4], antidiag), GenP([16,16], antidiag))"),
    "rev_3d": "GroupBy([4,6,5]).OrderBy(GenP([4,6,5], identity)).OrderBy(RegP([4,30],[2,1]))",
}

BIG_DSL = [
    ("cfg1_tiled_4096", "GroupBy([4096,4096]).OrderBy(RegP([128,32,128,32],[1,3,2,4]))",
     "reference"),
    ("cfg2_transpose_16384", "GroupBy([16384,16384]).OrderBy(Col(16384,16384))", "emitted"),
    ("cfg4_antidiag_16384", "GroupBy([16384,16384]).OrderBy(GenP([16384,16384], antidiag))",
     "emitted"),
]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    args = ap.parse_args()
    rng = random.Random(20261017)
    cases = []
    print("small layouts", flush=True)
    for name, dsl in SMALL_DSL.items():
        cases.append(small_case(name, lego.parse_layout(dsl), dsl))
    from helpers import layout_corpus  # the reference test-suite's corpus
    for k, g in enumerate(layout_corpus(seed=20240901, count=30, max_elems=40_000)):
        cases.append(small_case(f"corpus_{k:02d}", g))
    print("bench layouts", flush=True)
    for name, dsl, full in BIG_DSL:
        if args.quick and full == "emitted":
            full = None
        cases.append(big_case(name, dsl, full, rng))
    doc = {"generator": "tests/golden/make_golden.py", "reference": "/root/reference/pkg/src/lego",
           "reference_version": lego.__version__, "cases": cases}
    with open(OUT, "w") as fh:
        json.dump(doc, fh, separators=(",", ":"))
    print(f"wrote {OUT} ({os.path.getsize(OUT) / 1e6:.1f} MB, {len(cases)} cases)")


if __name__ == "__main__":
    main()
