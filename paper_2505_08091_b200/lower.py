"""Lowering of layouts to kernel plans (the step between the algebra and CUDA).

Builds the index expressions the kernels need directly from the layout's own
``apply``/``inv`` (reference ``layout.py:313-328``), composing stage by stage
on *flat* positions so that the canonical flatten/unflatten pair around the
logical index cancels instead of surviving as div/mod chains, then picks the
kernel family by *proving* structural facts about the simplified map:

* ``contiguous_width`` -- g(w*q + r) - g(w*q) - r simplifies to 0, i.e. every
  aligned run of w destination elements reads w consecutive source elements
  (16-byte vector loads are then exact);
* ``digit_terms`` -- g is a permutation of mixed-radix digits of f
  (``sum(((f // lo) % span) * stride)`` with the digit ranges tiling
  ``[1, n)``), which licenses the register-tiled transpose: the tile geometry
  and the tile-origin function are derived from the digits.

Everything here is host-side and runs once per (layout pair, element size);
the results are cached by :mod:`.kernels`.
"""

from __future__ import annotations

import math
from typing import Dict, List, Optional, Tuple

from .errors import ArityMismatch, ShapeMismatch
from .expr import (
    Add,
    And,
    Call,
    Cmp,
    Expr,
    FloorDiv,
    IntConst,
    Mod,
    Mul,
    Select,
    Sub,
    Var,
    VarRange,
    as_expr,
)
from .layout import ExpandBy, GroupBy, canon_flatten, canon_unflatten
from .simplify import Intervals, _digit_of, _lin_of, simplify


def substitute(e: Expr, env: Dict[str, Expr]) -> Expr:
    """Replace variables by expressions (DAG-aware, memoised)."""
    memo: Dict[Expr, Expr] = {}

    def sub(n):
        got = memo.get(n)
        if got is not None:
            return got
        t = type(n)
        if t is Var:
            out = env.get(n.name, n)
        elif t is IntConst:
            out = n
        elif t in (Add, Sub, Mul):
            out = t(sub(n.lhs), sub(n.rhs))
        elif t in (FloorDiv, Mod):
            out = t(sub(n.num), sub(n.den))
        elif t is Select:
            out = Select(cond(n.cond), sub(n.then), sub(n.orelse))
        elif t is Call:
            out = Call(n.intrinsic, tuple(sub(a) for a in n.args))
        else:
            raise TypeError(n)
        memo[n] = out
        return out

    def cond(c):
        if type(c) is Cmp:
            return Cmp(c.op, sub(c.lhs), sub(c.rhs))
        return And(cond(c.lhs), cond(c.rhs))

    return sub(e)


# ---------------------------------------------------------------------------
# Flat maps.
# ---------------------------------------------------------------------------

def _group(layout):
    return layout.inner if isinstance(layout, ExpandBy) else layout


def logical_size(layout) -> int:
    return math.prod(layout.dims)


def physical_size(layout) -> int:
    return layout.size


def apply_flat(layout, x: Expr) -> Expr:
    """Position of the logical element whose row-major flat index is x:
    ``layout.apply(canon_unflatten(dims, x))`` with the leading
    flatten(unflatten(x)) = x cancelled."""
    g = _group(layout)
    g._check()
    pos = x
    for stage in g.orders:
        pos = stage.apply(canon_unflatten(stage.dims, pos))
    if isinstance(layout, ExpandBy):
        layout._check()
        coords = canon_unflatten(layout.expanded, pos)
        phys = canon_flatten(layout.physical, coords, check=False)
        from .expr import and_all, lt
        pos = Select(and_all(lt(c, n) for c, n in zip(coords, layout.physical)), phys,
                     IntConst(-1))
    return pos


def inv_flat(layout, f: Expr) -> Expr:
    """Row-major flat logical index of the element at position f:
    ``canon_flatten(dims, layout.inv(f))`` with the trailing pair cancelled."""
    pos = f
    if isinstance(layout, ExpandBy):
        layout._check()
        pos = canon_flatten(layout.expanded, canon_unflatten(layout.physical, pos), check=False)
    g = _group(layout)
    if g.injective:
        from .errors import LegoError
        raise LegoError("injective layout exports apply only, not inv")
    g._check()
    for stage in g.orders[::-1]:
        pos = canon_flatten(stage.dims, stage.inv(pos), check=False)
    return pos


def flat_var(name: str, n: int) -> Var:
    return Var(name, VarRange(0, n))


def apply_map_expr(layout) -> Tuple[Var, Expr]:
    x = flat_var("x", logical_size(layout))
    return x, simplify(as_expr(apply_flat(layout, x)))


def inv_map_expr(layout) -> Tuple[Var, Expr]:
    f = flat_var("f", physical_size(layout))
    return f, simplify(as_expr(inv_flat(layout, f)))


def check_pair(src_layout, dst_layout):
    if src_layout is None and dst_layout is None:
        raise ShapeMismatch("remap needs at least one layout")
    if src_layout is not None and dst_layout is not None:
        if tuple(src_layout.dims) != tuple(dst_layout.dims):
            raise ArityMismatch(f"source layout dims {tuple(src_layout.dims)} differ from "
                                f"destination dims {tuple(dst_layout.dims)}")


def gather_expr(src_layout, dst_layout) -> Tuple[Var, Expr, int, int]:
    """g with dst[f] = src[g(f)]: g = src.apply o dst.inv (row-major where a
    side is None).  Returns (f, g, dst size, src size)."""
    check_pair(src_layout, dst_layout)
    some = src_layout if src_layout is not None else dst_layout
    n_dst = physical_size(dst_layout) if dst_layout is not None else logical_size(some)
    n_src = physical_size(src_layout) if src_layout is not None else logical_size(some)
    f = flat_var("f", n_dst)
    x = inv_flat(dst_layout, f) if dst_layout is not None else f
    s = apply_flat(src_layout, as_expr(x)) if src_layout is not None else x
    return f, simplify(as_expr(s)), n_dst, n_src


# ---------------------------------------------------------------------------
# Structural proofs.
# ---------------------------------------------------------------------------

def contiguous_width(g: Expr, f: Var, n: int, widths=(16, 8, 4, 2)) -> int:
    """Largest w in widths such that g(w*q + r) == g(w*q) + r for all q, r."""
    for w in widths:
        if n % w:
            continue
        q = Var("q", VarRange(0, n // w))
        r = Var("r", VarRange(0, w))
        lhs = substitute(g, {f.name: q * w + r})
        rhs = substitute(g, {f.name: q * w})
        if simplify(lhs - rhs - r) == IntConst(0):
            return w
    return 1


def digit_terms(g: Expr, f: Var, n: int) -> Optional[List[Tuple[int, int, int]]]:
    """If g == sum(((f // lo) % span) * stride) with digit runs tiling [1, n),
    return [(lo, span, stride)] sorted by lo; else None."""
    lin = _lin_of(g)
    if lin.const != 0:
        return None
    digits = []
    for atom, coef in lin.terms.items():
        base, lo, span = _digit_of(atom)
        if base is None or base != f:
            return None
        if span is None:
            if n % lo:
                return None
            span = n // lo
        digits.append((lo, span, coef))
    digits.sort()
    expect = 1
    for lo, span, _ in digits:
        if lo != expect:
            return None
        expect = lo * span
    if expect != n:
        return None
    return digits


def split_digit(digits, lo_target: int, inner: int):
    """Split the digit at lo_target into (inner) and (span // inner) parts."""
    out = []
    for lo, span, stride in digits:
        if lo == lo_target and span > inner:
            out.append((lo, inner, stride))
            out.append((lo * inner, span // inner, stride * inner))
        else:
            out.append((lo, span, stride))
    return out


class TransposePlan:
    def __init__(self, tiles: int, sx: int, dy: int, origin_f0: Expr, origin_s0: Expr, t: Var,
                 tx: int, ty: int):
        self.tiles, self.sx, self.dy = tiles, sx, dy
        self.origin_f0, self.origin_s0, self.t = origin_f0, origin_s0, t
        self.tx, self.ty = tx, ty


def transpose_plan(g: Expr, f: Var, n: int, elem_bytes: int, x_vectors: int = 4,
                   y_vectors: int = 8, tile_order: str = "x") -> Optional[TransposePlan]:
    """Warp-tiled transpose geometry for a digit-permutation gather: a warp
    tile is (x_vectors*V) x (y_vectors*V) elements, V = 16 / elem_bytes."""
    if 16 % elem_bytes:
        return None
    digits = digit_terms(g, f, n)
    if digits is None:
        return None
    v = 16 // elem_bytes
    tx, ty = x_vectors * v, y_vectors * v   # x along the dst digit, y along the src digit
    x_lo, x_span, sx = digits[0]
    if sx == 1:
        return None                        # contiguous: the gather path is better
    ydig = [d for d in digits if d[2] == 1]
    if len(ydig) != 1:
        return None
    y_lo, y_span, _ = ydig[0]
    if x_span % tx or y_span % ty or sx % v:
        return None
    # every other digit must keep 16-byte alignment on both sides
    for lo, span, stride in digits:
        if (lo, span) in ((x_lo, x_span), (y_lo, y_span)):
            continue
        if stride % v or lo % v:
            return None
    # tile index t -> tile coordinates -> dst origin f0.  The walk order is a
    # LEGO layout over the tile grid (x_hi, mid, y_hi, hi):
    #   "x": x_hi fastest (concurrent warps sweep dst rows),
    #   "y": y_hi fastest (concurrent warps sweep src rows),
    #   "block": 8 x 8 tile blocks, x fastest inside a block (both sides local)
    x_hi = x_span // tx
    mid = y_lo // x_span
    y_hi = y_span // ty
    hi = n // (y_lo * y_span)
    tiles = x_hi * mid * y_hi * hi
    t = Var("t", VarRange(0, tiles))
    order = tile_order
    if order == "block" and (x_hi % 8 or y_hi % 8):
        order = "x"
    if order == "y":
        c2 = t % y_hi
        c0 = (t // y_hi) % x_hi
        c1 = (t // (y_hi * x_hi)) % mid
        c3 = t // (y_hi * x_hi * mid)
    elif order == "block":
        lx = t % 8
        ly = (t // 8) % 8
        gx = (t // 64) % (x_hi // 8)
        gy = (t // (64 * (x_hi // 8))) % (y_hi // 8)
        rest = t // (x_hi * y_hi)
        c0 = gx * 8 + lx
        c2 = gy * 8 + ly
        c1 = rest % mid
        c3 = rest // mid
    else:
        c0 = t % x_hi
        c1 = (t // x_hi) % mid
        c2 = (t // (x_hi * mid)) % y_hi
        c3 = t // (x_hi * mid * y_hi)
    f0 = simplify(c0 * tx + c1 * x_span + c2 * (ty * y_lo) + c3 * (y_lo * y_span))
    s0 = simplify(substitute(g, {f.name: f0}))
    return TransposePlan(tiles, sx, y_lo, f0, s0, t, tx, ty)


def antidiag_side(layout) -> Optional[int]:
    """n if the layout is GroupBy([n, n]).OrderBy(GenP([n, n], antidiag))."""
    from .layout import GenP
    if not isinstance(layout, GroupBy) or layout.injective or len(layout.tiles) != 1:
        return None
    if len(layout.orders) != 1 or len(layout.orders[0].perms) != 1:
        return None
    p = layout.orders[0].perms[0]
    if not isinstance(p, GenP) or p.name != "antidiag" or len(p.shape) != 2:
        return None
    n = p.shape[0]
    if tuple(layout.dims) != (n, n):
        return None
    return n


def diagonal_runs_contiguous(layout, n: int) -> bool:
    """Prove pos(i+1, t-i-1) == pos(i, t-i) + 1 on every anti-diagonal t."""
    # the layout is one GenP over its whole logical shape, so on in-range
    # coordinates apply == the GenP's own symbolic fwd (layout.py:187-191)
    p = layout.orders[0].perms[0]
    i = Var("i", VarRange(0, n - 1))
    t = Var("t", VarRange(0, 2 * n - 1))
    a = p.fwd.symbolic((i + 1, t - i - 1))
    b = p.fwd.symbolic((i, t - i))
    return simplify(as_expr(a) - as_expr(b) - 1) == IntConst(0)


def value_range(e: Expr):
    return Intervals().of(e)


def value_at(e: Expr, x: Var, v: int) -> Optional[int]:
    """e with x = v, if it folds to a constant."""
    got = simplify(substitute(e, {x.name: IntConst(v)}))
    return got.value if type(got) is IntConst else None


class NarrowPlan:
    """Register interleave of a digit permutation whose innermost digit on one
    side spans less than a 16-byte vector (AoS <-> SoA style), V = 16/E:

    * mode 1 -- the source-innermost digit y is small (Y | V, Y < V) and the
      destination-innermost digit x follows it in the source (source stride
      Y): a lane loads one 16-byte source vector = P = V/Y consecutive x
      values x Y, and stores Y chunks of P elements, chunk y at destination
      ``gen::map(s + y)`` (the inverse digit permutation, contiguous in x);
    * mode 2 -- the destination-innermost digit x is small (Xd | V, Xd < V)
      and the source-innermost digit y follows it in the destination: a lane
      loads Xd chunks of P = V/Xd elements, chunk x from source
      ``gen::map(f + x)`` (the gather map), and stores one 16-byte vector.

    A warp covers 32*V consecutive source (mode 1) / destination (mode 2)
    elements; ``small`` is Y / Xd."""

    def __init__(self, mode, small, var, fmap):
        self.mode, self.small, self.var, self.map = mode, small, var, fmap


def narrow_plan(g: Expr, f: Var, n: int, elem_bytes: int) -> Optional[NarrowPlan]:
    """Prove the NarrowPlan conditions on the digit decomposition of g and
    build the per-chunk address map; None when they do not hold."""
    if 16 % elem_bytes:
        return None
    v = 16 // elem_bytes
    if n % (32 * v):
        return None
    digits = digit_terms(g, f, n)                # (dst lo, span, src stride), dst-innermost first
    if digits is None or len(digits) < 2:
        return None
    x_lo, x_span, sx = digits[0]
    ydig = [d for d in digits if d[2] == 1]
    if len(ydig) != 1:
        return None
    y_lo, y_span, _ = ydig[0]
    cand1 = y_span < v and v % y_span == 0 and sx == y_span and x_span % (v // y_span) == 0
    cand2 = x_span < v and v % x_span == 0 and y_lo == x_span and y_span % (v // x_span) == 0 and sx != 1
    if cand1 and cand2 and x_span < y_span:
        cand1 = False                            # prefer the mode with the larger chunks
    if cand1 and (v // y_span) * elem_bytes < 4:
        cand1 = False                            # chunks below 4 bytes: not worth it
    if cand2 and (v // x_span) * elem_bytes < 4:
        cand2 = False
    if cand1:
        mode, small = 1, y_span
        p = v // small
        # chunks start at x multiples of P; every other digit keeps them P-aligned in the destination
        if any(lo % p for lo, span, stride in digits if (lo, span, stride) != digits[0]):
            return None
        s = Var("s", VarRange(0, n))
        h = IntConst(0)                          # inverse digit permutation: destination of source s
        for lo, span, stride in digits:
            h = h + ((s // stride) % span) * lo if stride > 1 else h + (s % span) * lo
        return NarrowPlan(1, small, s, simplify(as_expr(h)))
    if cand2:
        mode, small = 2, x_span
        p = v // small
        if any(stride % p for lo, span, stride in digits if (lo, span, stride) != ydig[0]):
            return None
        return NarrowPlan(2, small, f, g)
    return None
