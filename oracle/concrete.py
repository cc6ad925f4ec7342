"""Concrete-callable oracle for layouts with user-defined permutations --
TEST INFRASTRUCTURE ONLY (see oracle.py's header for who may import it).

The reference semantics of a user bijection is its own concrete callable
(``PermFn.concrete``; ``GenP.apply`` / ``GenP.inv``, reference
``pkg/src/lego/layout.py:187-200``): the symbolic builder is only the
route to code generation and may disagree with it.  The C oracle knows the
built-in permutations only, so parity of layouts holding arbitrary ``GenP``s
is checked here, by evaluating the reference algorithm over whole index
spaces with the concrete callables:

* ``GroupBy.apply`` (layout.py:313-318): canonical flatten, then every
  ``OrderBy`` stage in listed order -- unflatten into the stage's dims, each
  permutation on its coordinates, mixed-radix recombination outermost-first
  (layout.py:237-246);
* ``GroupBy.inv`` (layout.py:320-328): stages in reverse, each peeling its
  permutations innermost-first with % and // (layout.py:248-258);
* ``RegP`` (layout.py:142-149): flatten the sigma-permuted index in the
  sigma-permuted shape, and back;
* ``ExpandBy`` (layout.py:383-400): masked positions are -1.

Layout objects are read structurally (``tiles``, ``orders``, ``perms``,
``shape``, ``sigma``, ``fwd.concrete``, ``inv_fn.concrete``), so the same
code evaluates the reference's own objects and the backend's mirror of them.
A ``GenP`` callable is first tried on whole numpy coordinate arrays (most
index arithmetic -- ``//``, ``%``, ``^``, ``>>`` -- is elementwise with
Python's floor semantics); the vectorised result is accepted only if it
matches scalar calls on a spread sample, otherwise the callable is applied
element by element on a fork pool of all host cores.
"""

from __future__ import annotations

import math
import multiprocessing as mp
import os
from typing import Sequence

import numpy as np

SAMPLE = 512          # scalar calls that must agree with a vectorised evaluation


def _unflatten(shape: Sequence[int], flat: np.ndarray):
    out = []
    for n in reversed(shape[1:]):
        out.append(flat % n)
        flat = flat // n
    out.append(flat)
    return out[::-1]


def _flatten(shape: Sequence[int], coords) -> np.ndarray:
    acc = np.zeros_like(coords[0])
    for c, n in zip(coords, shape):
        acc = acc * n + c
    return acc


# ---------------------------------------------------------------------------
# concrete callables over arrays
# ---------------------------------------------------------------------------

_POOL_FN = None


def _pool_chunk(args):
    rows, fwd = args
    fn = _POOL_FN
    if fwd:
        return np.asarray([fn(tuple(int(v) for v in r)) for r in rows], dtype=np.int64)
    res = [fn(int(r)) for r in rows]
    return np.asarray([tuple(int(c) for c in (x if isinstance(x, (tuple, list)) else (x,))) for x in res],
                      dtype=np.int64)


def _threaded() -> bool:
    """fork() is unsafe once CUDA (and its threads) is up in this process."""
    import sys
    torch = sys.modules.get("torch")
    return bool(torch is not None and torch.cuda.is_available() and torch.cuda.is_initialized())


def _scalar_map(fn, inputs: np.ndarray, fwd: bool) -> np.ndarray:
    """fn applied element by element (fork pool for large inputs)."""
    global _POOL_FN
    n = len(inputs)
    if n <= 1 << 14 or not hasattr(os, "fork") or _threaded():
        _POOL_FN = fn
        return _pool_chunk((inputs, fwd))
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    chunks = np.array_split(inputs, max(1, cores * 4))
    _POOL_FN = fn
    with mp.get_context("fork").Pool(cores) as pool:
        parts = pool.map(_pool_chunk, [(c, fwd) for c in chunks])
    return np.concatenate(parts)


def _sample_idx(n: int) -> np.ndarray:
    return np.unique(np.linspace(0, n - 1, num=min(n, SAMPLE)).astype(np.int64)) if n else np.zeros(0, np.int64)


def genp_apply(p, coords) -> np.ndarray:
    """GenP.apply over arrays of coordinates: fwd.concrete((c0, c1, ...))."""
    fn = p.fwd.concrete
    n = len(coords[0])
    try:
        got = np.asarray(fn(tuple(coords)), dtype=np.int64)
        if got.shape != (n,):
            raise ValueError("not elementwise")
        s = _sample_idx(n)
        want = np.asarray([fn(tuple(int(c[k]) for c in coords)) for k in s], dtype=np.int64)
        if np.array_equal(got[s], want):
            return got
    except Exception:  # noqa: BLE001 - fall back to scalar calls
        pass
    return _scalar_map(fn, np.stack(coords, axis=1), True)


def genp_inv(p, flat: np.ndarray):
    """GenP.inv over an array of flat indices: inv_fn.concrete(flat)."""
    if p.inv_fn is None:
        raise ValueError("permutation has no inverse (injective mode)")
    fn = p.inv_fn.concrete
    d = len(p.shape)
    n = len(flat)
    try:
        got = fn(flat)
        got = [np.asarray(c, dtype=np.int64) for c in (got if isinstance(got, (tuple, list)) else (got,))]
        if len(got) != d or any(c.shape != (n,) for c in got):
            raise ValueError("not elementwise")
        s = _sample_idx(n)
        for k in s:
            want = fn(int(flat[k]))
            want = tuple(want) if isinstance(want, (tuple, list)) else (want,)
            if tuple(int(c[k]) for c in got) != tuple(int(w) for w in want):
                raise ValueError("vectorised evaluation disagrees")
        return got
    except Exception:  # noqa: BLE001
        pass
    rows = _scalar_map(fn, flat, False)
    return [rows[:, k] for k in range(d)]


def _perm_apply(p, coords) -> np.ndarray:
    if hasattr(p, "sigma"):                                   # RegP
        s = p.sigma
        return _flatten([p.shape[k - 1] for k in s], [coords[k - 1] for k in s])
    return genp_apply(p, coords)


def _perm_inv(p, flat: np.ndarray):
    if hasattr(p, "sigma"):                                   # RegP
        s = p.sigma
        permuted = _unflatten([p.shape[k - 1] for k in s], flat)
        out = [None] * len(s)
        for pos, k in enumerate(s):
            out[k - 1] = permuted[pos]
        return out
    return genp_inv(p, flat)


# ---------------------------------------------------------------------------
# layouts over whole index ranges
# ---------------------------------------------------------------------------

def _group(layout):
    return layout.inner if hasattr(layout, "expanded") else layout


def dims(layout):
    return tuple(n for t in _group(layout).tiles for n in t)


def logical_size(layout) -> int:
    return math.prod(dims(layout))


def physical_size(layout) -> int:
    if hasattr(layout, "expanded"):
        return math.prod(layout.physical)
    return logical_size(layout)


def apply_all(layout, first: int = 0, count=None) -> np.ndarray:
    """positions[k] = layout.apply(canon_unflatten(dims, first + k)), -1 where masked."""
    n = logical_size(layout)
    count = n - first if count is None else count
    pos = np.arange(first, first + count, dtype=np.int64)
    for stage in _group(layout).orders:
        sd = [d for p in stage.perms for d in p.shape]
        coords = _unflatten(sd, pos)
        acc = None
        k = 0
        for p in stage.perms:
            r = len(p.shape)
            sub = _perm_apply(p, coords[k:k + r])
            k += r
            acc = sub if acc is None else acc * math.prod(p.shape) + sub
        pos = acc
    if hasattr(layout, "expanded"):
        c = _unflatten(layout.expanded, pos)
        ok = np.ones(len(pos), dtype=bool)
        for a, b in zip(c, layout.physical):
            ok &= a < b
        pos = np.where(ok, _flatten(layout.physical, [np.minimum(a, b - 1) for a, b in zip(c, layout.physical)]),
                       -1)
    return pos


def inv_all(layout, first: int = 0, count=None) -> np.ndarray:
    """logical[k] = canon_flatten(dims, layout.inv(first + k))."""
    n = physical_size(layout)
    count = n - first if count is None else count
    pos = np.arange(first, first + count, dtype=np.int64)
    if hasattr(layout, "expanded"):
        pos = _flatten(layout.expanded, _unflatten(layout.physical, pos))
    for stage in _group(layout).orders[::-1]:
        out = []
        flat = pos
        for p in stage.perms[::-1]:
            radix = math.prod(p.shape)
            out = list(_perm_inv(p, flat % radix)) + out
            flat = flat // radix
        pos = _flatten([d for p in stage.perms for d in p.shape], out)
    return pos


def remap(src: np.ndarray, src_layout, dst_layout, dst_size=None) -> np.ndarray:
    """dst[dst.apply(x)] = src[src.apply(x)] for every logical x (None =
    row-major over the other side's dims); unwritten positions stay 0."""
    some = src_layout if src_layout is not None else dst_layout
    n = logical_size(some)
    s = apply_all(src_layout) if src_layout is not None else np.arange(n, dtype=np.int64)
    d = apply_all(dst_layout) if dst_layout is not None else np.arange(n, dtype=np.int64)
    if dst_size is None:
        dst_size = physical_size(dst_layout) if dst_layout is not None else n
        if dst_layout is not None and getattr(_group(dst_layout), "injective", False):
            dst_size = int(d.max()) + 1 if len(d) else 0
    out = np.zeros(dst_size, dtype=src.dtype)
    keep = (s >= 0) & (d >= 0)
    out[d[keep]] = src[s[keep]]
    return out
