"""CPU oracle for the B200 backend -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this module, and
only as the *checker* or the timed CPU baseline -- never as the thing
measured or shipped.  The product package never imports it.

It restates the reference algorithm (``/root/reference/pkg/src/lego``) for
the hot path -- per-element ``GroupBy.apply`` / ``inv`` (``layout.py:313-328``)
and everything below it -- in plain C (``lego_oracle.c``, built into
``oracle/liblego_oracle.so`` by ``oracle/Makefile``), driven by a layout
*spec* that this module parses from the layout DSL with its own small parser
(independent of the product's ``dsl.py``), or receives as JSON from the
golden fixtures.  Pinning: ``tests/test_oracle.py`` checks it against the
vectors ``tests/golden/make_golden.py`` produced by running the reference.

Also here: float64 / fp32 restatements for the kernels the reference does
not ship (row softmax, bf16 GEMM; "parity unpinned" for those -- there is
no reference implementation to pin them to) and the NW DP.
"""

from __future__ import annotations

import ctypes
import json
import math
import os
import re
import subprocess
from typing import List, Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liblego_oracle.so")
MAGIC = 0x4C45474F
KIND = {"regp": 0, "identity": 1, "rev": 2, "antidiag": 3}

_lib = None


def build(force: bool = False) -> str:
    src = os.path.join(HERE, "lego_oracle.c")
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(src):
        subprocess.check_call(["make", "-s", "-C", HERE])
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = ctypes.CDLL(LIB_PATH)
        i64p = ctypes.POINTER(ctypes.c_int64)
        for name in ("oracle_apply_range", "oracle_inv_range"):
            fn = getattr(L, name)
            fn.argtypes = [i64p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, i64p]
            fn.restype = ctypes.c_int
        L.oracle_remap.argtypes = [i64p, ctypes.c_int64, i64p, ctypes.c_int64, ctypes.c_int64,
                                   ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
                                   ctypes.c_int64, ctypes.c_int64]
        L.oracle_remap.restype = ctypes.c_int
        i32p = ctypes.POINTER(ctypes.c_int32)
        for name in ("oracle_nw", "oracle_nw_rowmajor"):
            fn = getattr(L, name)
            fn.argtypes = [i32p, ctypes.c_int64, ctypes.c_int32, i32p]
            fn.restype = ctypes.c_int
        L.oracle_threads.restype = ctypes.c_int
        L.oracle_set_threads.argtypes = [ctypes.c_int]
        L.oracle_set_threads.restype = None
        _lib = L
    return _lib


def threads() -> int:
    return lib().oracle_threads()


def set_threads(n: int) -> None:
    lib().oracle_set_threads(int(n))


# ---------------------------------------------------------------------------
# Layout specs: a plain-dict description and the DSL parser that makes one.
# ---------------------------------------------------------------------------

def _regp(shape, sigma):
    return {"kind": "regp", "shape": list(shape), "sigma": list(sigma)}


def _sigma_tile(d, q):
    return [k + 1 + d * h for k in range(d) for h in range(q)]


_TOK = re.compile(r"\s*([A-Za-z_]\w*|\d+|[()\[\],.])")


class _P:
    def __init__(self, text):
        self.t = []
        pos = 0
        text = text.strip()
        while pos < len(text):
            m = _TOK.match(text, pos)
            if not m:
                raise ValueError(f"oracle parser: bad input at {pos}")
            self.t.append(m.group(1))
            pos = m.end()
            while pos < len(text) and text[pos].isspace():
                pos += 1
        self.k = 0

    def nxt(self):
        tok = self.t[self.k]
        self.k += 1
        return tok

    def eat(self, s):
        tok = self.nxt()
        if tok != s:
            raise ValueError(f"oracle parser: expected {s}, got {tok}")

    def peek(self):
        return self.t[self.k] if self.k < len(self.t) else None

    def ints(self):
        vals = [int(self.nxt())]
        while self.peek() == ",":
            self.nxt()
            vals.append(int(self.nxt()))
        return vals

    def shape(self):
        self.eat("[")
        v = self.ints()
        self.eat("]")
        return v

    def many(self, fn):
        out = [fn()]
        while self.peek() == ",":
            self.nxt()
            out.append(fn())
        return out

    def perm(self):
        w = self.nxt()
        self.eat("(")
        if w == "RegP":
            shape = self.shape()
            self.eat(",")
            p = _regp(shape, self.shape())
        elif w == "GenP":
            shape = self.shape()
            self.eat(",")
            name = self.nxt()
            kind = {"identity": "identity", "rev1d": "rev", "rev2d": "rev",
                    "antidiag": "antidiag"}[name]
            p = {"kind": kind, "shape": shape}
        elif w in ("Row", "Col"):
            ext = self.shape() if self.peek() == "[" else self.ints()
            if w == "Row":
                p = _regp(ext, range(1, len(ext) + 1))
            else:
                p = _regp(ext[::-1], range(len(ext), 0, -1))
        else:
            raise ValueError(f"oracle parser: unknown perm {w}")
        self.eat(")")
        return p

    def layout(self):
        w = self.nxt()
        self.eat("(")
        if w == "GroupBy":
            spec = {"kind": "group", "tiles": self.many(self.shape), "stages": []}
        elif w == "TileBy":
            tiles = self.many(self.shape)
            cat = [n for t in tiles for n in t]
            spec = {"kind": "group", "tiles": tiles,
                    "stages": [[_regp(cat, _sigma_tile(len(tiles[0]), len(tiles)))]]}
        elif w == "TileOrderBy":
            perms = self.many(self.perm)
            permuted = [p["shape"][s - 1] for p in perms for s in p["sigma"]]
            spec = {"kind": "group", "tiles": [p["shape"] for p in perms],
                    "stages": [perms, [_regp(permuted, _sigma_tile(len(perms[0]["shape"]),
                                                                  len(perms)))]]}
        elif w == "ExpandBy":
            phys = self.shape()
            self.eat(",")
            expd = self.shape()
            self.eat(",")
            inner = self.layout()
            spec = {"kind": "expand", "physical": phys, "expanded": expd, "inner": inner}
        else:
            raise ValueError(f"oracle parser: unknown layout {w}")
        self.eat(")")
        while self.peek() == ".":
            self.nxt()
            if self.nxt() != "OrderBy":
                raise ValueError("oracle parser: only OrderBy chains")
            self.eat("(")
            spec["stages"].append(self.many(self.perm))
            self.eat(")")
        return spec


def parse(text: str) -> dict:
    p = _P(text)
    spec = p.layout()
    if p.peek() is not None:
        raise ValueError("oracle parser: trailing input")
    return spec


def dims(spec) -> List[int]:
    if spec["kind"] == "expand":
        return dims(spec["inner"])
    return [n for t in spec["tiles"] for n in t]


def size(spec) -> int:
    if spec["kind"] == "expand":
        return math.prod(spec["physical"])
    return math.prod(dims(spec))


def logical_size(spec) -> int:
    return math.prod(dims(spec))


def encode(spec) -> np.ndarray:
    out = [MAGIC, 1]
    if spec["kind"] == "expand":
        out += [1, len(spec["physical"])] + list(spec["physical"]) + list(spec["expanded"])
        g = spec["inner"]
    else:
        out += [0]
        g = spec
    d = dims(g)
    out += [len(d)] + d + [len(g["stages"])]
    for stage in g["stages"]:
        out.append(len(stage))
        for p in stage:
            out += [KIND[p["kind"]], len(p["shape"])] + list(p["shape"])
            if p["kind"] == "regp":
                out += list(p["sigma"])
    return np.asarray(out, dtype=np.int64)


def _ptr(a, ct=ctypes.c_int64):
    return a.ctypes.data_as(ctypes.POINTER(ct))


# ---------------------------------------------------------------------------
# Bulk evaluation through the C restatement.
# ---------------------------------------------------------------------------

def apply_range(spec, first: int = 0, count: Optional[int] = None) -> np.ndarray:
    """out[k] = apply(unflatten(dims, first + k)) (-1 = ExpandBy mask)."""
    if count is None:
        count = logical_size(spec) - first
    desc = encode(spec)
    out = np.empty(count, dtype=np.int64)
    rc = lib().oracle_apply_range(_ptr(desc), desc.size, first, count, _ptr(out))
    if rc:
        raise ValueError(f"oracle descriptor rejected ({rc})")
    return out


def inv_range(spec, first: int = 0, count: Optional[int] = None) -> np.ndarray:
    """out[k] = canon_flatten(dims, inv(first + k))."""
    if count is None:
        count = size(spec) - first
    desc = encode(spec)
    out = np.empty(count, dtype=np.int64)
    rc = lib().oracle_inv_range(_ptr(desc), desc.size, first, count, _ptr(out))
    if rc:
        raise ValueError(f"oracle descriptor rejected ({rc})")
    return out


def remap(src: np.ndarray, src_spec, dst_spec, dst_size: Optional[int] = None,
          first: int = 0, count: Optional[int] = None, out: Optional[np.ndarray] = None):
    """dst[dst.apply(x)] = src[src.apply(x)] for logical x (None = row-major)."""
    some = src_spec or dst_spec
    n = logical_size(some)
    if count is None:
        count = n - first
    if out is None:
        out = np.zeros(dst_size if dst_size is not None else (size(dst_spec) if dst_spec else n),
                       dtype=src.dtype)
    ds = encode(src_spec) if src_spec else np.zeros(1, np.int64)
    dd = encode(dst_spec) if dst_spec else np.zeros(1, np.int64)
    src = np.ascontiguousarray(src)
    rc = lib().oracle_remap(_ptr(ds), ds.size if src_spec else 0, _ptr(dd),
                            dd.size if dst_spec else 0, n,
                            src.ctypes.data, out.ctypes.data, src.dtype.itemsize, first, count)
    if rc:
        raise ValueError(f"oracle descriptor rejected ({rc})")
    return out


def nw(sim: np.ndarray, penalty: int, rowmajor: bool = False) -> np.ndarray:
    """Needleman-Wunsch score matrix (n+1)^2 for an n x n int32 similarity."""
    sim = np.ascontiguousarray(sim, dtype=np.int32)
    n = sim.shape[0]
    score = np.empty((n + 1, n + 1), dtype=np.int32)
    fn = lib().oracle_nw_rowmajor if rowmajor else lib().oracle_nw
    fn(_ptr(sim, ctypes.c_int32), n, penalty, _ptr(score, ctypes.c_int32))
    return score


# ---------------------------------------------------------------------------
# Pure-Python scalar restatement (small cases; used to cross-check the C).
# ---------------------------------------------------------------------------

def _unflat(shape, f):
    out = []
    for n in reversed(shape[1:]):
        out.append(f % n)
        f //= n
    out.append(f)
    return out[::-1]


def _flat(shape, idx):
    acc = 0
    for c, n in zip(idx, shape):
        acc = acc * n + c
    return acc


def _perm_apply(p, idx):
    shape = p["shape"]
    if p["kind"] == "regp":
        s = p["sigma"]
        return _flat([shape[k - 1] for k in s], [idx[k - 1] for k in s])
    if p["kind"] == "identity":
        return _flat(shape, idx)
    if p["kind"] == "rev":
        return _flat(shape, [n - 1 - c for c, n in zip(idx, shape)])
    n = shape[0]
    i, j = idx
    t = i + j + 1
    if t <= n:
        return i + t * (t - 1) // 2
    t = 2 * n - t
    return n * n - n + i - t * (t - 1) // 2


def py_apply(spec, idx) -> Optional[int]:
    g = spec["inner"] if spec["kind"] == "expand" else spec
    flat = _flat(dims(g), idx)
    for stage in g["stages"]:
        sd = [n for p in stage for n in p["shape"]]
        c = _unflat(sd, flat)
        acc, pos = 0, 0
        for p in stage:
            r = len(p["shape"])
            acc = acc * math.prod(p["shape"]) + _perm_apply(p, c[pos:pos + r])
            pos += r
        flat = acc
    if spec["kind"] == "expand":
        c = _unflat(spec["expanded"], flat)
        if any(a >= b for a, b in zip(c, spec["physical"])):
            return None
        return _flat(spec["physical"], c)
    return flat


# ---------------------------------------------------------------------------
# Float restatements (no reference implementation exists: parity unpinned).
# ---------------------------------------------------------------------------

def softmax_rows_f64(x: np.ndarray) -> np.ndarray:
    x = x.astype(np.float64)
    m = x.max(axis=1, keepdims=True)
    e = np.exp(x - m)
    return e / e.sum(axis=1, keepdims=True)


def spec_from_json(text: str) -> dict:
    return json.loads(text)
