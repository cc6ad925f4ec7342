"""Golden vectors of user-defined GenPs, produced by RUNNING THE REFERENCE.

    python tests/golden/make_user_golden.py      (needs /root/reference; run here, not on the GPU box)

For every layout of tests/user_genps.py, built with the reference package
itself (``/root/reference/pkg/src/lego``), the reference's own per-element
``GroupBy.apply`` (layout.py:313-318) and ``GroupBy.inv`` (layout.py:320-328)
are evaluated over the WHOLE index space (a fork pool of all host cores);
the fixture keeps SHA-256 digests of the full tables (int64 little-endian)
plus 2048 sampled points in the clear.  tests/test_user_genps.py checks the
concrete-callable oracle (oracle/concrete.py) against it, which pins the
oracle that judges the CUDA path for arbitrary user bijections.
"""

import hashlib
import json
import math
import multiprocessing as mp
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(HERE))

import lego  # noqa: E402  (the reference)
from user_genps import FACTORIES  # noqa: E402

_LAYOUT = None


def _apply_chunk(bounds):
    lo, hi = bounds
    dims = _LAYOUT.dims
    out = np.empty(hi - lo, dtype=np.int64)
    for k, x in enumerate(range(lo, hi)):
        out[k] = _LAYOUT.apply(lego.canon_unflatten(dims, x))
    return out


def _inv_chunk(bounds):
    lo, hi = bounds
    dims = _LAYOUT.dims
    out = np.empty(hi - lo, dtype=np.int64)
    for k, f in enumerate(range(lo, hi)):
        out[k] = lego.canon_flatten(dims, _LAYOUT.inv(f))
    return out


def _table(fn, n):
    cores = len(os.sched_getaffinity(0))
    step = max(1, -(-n // (cores * 8)))
    chunks = [(lo, min(n, lo + step)) for lo in range(0, n, step)]
    with mp.get_context("fork").Pool(cores) as pool:
        return np.concatenate(pool.map(fn, chunks))


def main():
    global _LAYOUT
    cases = []
    rng = np.random.default_rng(7)
    for name, make in FACTORIES.items():
        _LAYOUT = make(lego)
        n = math.prod(_LAYOUT.dims)
        app = _table(_apply_chunk, n)
        case = {"name": name, "logical_size": n, "dims": list(_LAYOUT.dims),
                "injective": bool(_LAYOUT.injective),
                "apply_sha256": hashlib.sha256(app.astype("<i8").tobytes()).hexdigest()}
        xs = np.sort(rng.choice(n, size=2048, replace=False))
        case["samples"] = {"x": xs.tolist(), "apply": app[xs].tolist()}
        if not _LAYOUT.injective:
            inv = _table(_inv_chunk, n)
            case["inv_sha256"] = hashlib.sha256(inv.astype("<i8").tobytes()).hexdigest()
            case["samples"]["inv"] = inv[xs].tolist()
        cases.append(case)
        print(name, n, case["apply_sha256"][:12], flush=True)
    with open(os.path.join(HERE, "user_genps.json"), "w") as fh:
        json.dump({"generator": "tests/golden/make_user_golden.py", "reference": "/root/reference/pkg/src/lego",
                   "cases": cases}, fh)


if __name__ == "__main__":
    main()
