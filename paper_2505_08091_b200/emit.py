"""Expression printers and the target-profile plug-in point.

Mirrors reference ``pkg/src/lego/emit.py:33-102``: ``TargetProfile``,
``C_PROFILE`` / ``PYTHON_PROFILE`` / ``TRITON_PROFILE``, ``PROFILES``,
``get_profile``, ``RangeExpr``, ``emit_range`` and ``emit_expr`` with
``ranges=`` / ``broadcasts=``.  Printing is a pure structural walk with
minimal parentheses, so equal expressions print byte-identically.

New here: the ``cuda`` profile.  Unlike the C
profile, which prints floor division as ``/`` and silently assumes
non-negative operands (reference ``emit.py:4-7``), the CUDA profile proves
signs with interval analysis and prints ``lego_fdiv`` / ``lego_fmod`` (floor
semantics, defined in ``csrc/lego_index.cuh``) wherever a numerator may be
negative, and ``lego_isqrt`` (exact) for ``isqrt``.  Whole device functions
with CSE and typed temporaries come from :mod:`.codegen`; this printer is for
inline template splices.
"""

from __future__ import annotations

from typing import Mapping, Optional

from .errors import UnsupportedNode
from .expr import Add, And, Call, Cmp, Expr, FloorDiv, IntConst, Mod, Mul, Select, Sub, Var


class TargetProfile:
    __slots__ = ("name", "floordiv", "mod", "and_op", "select_style", "isqrt_name", "arange",
                 "paren_cmp_in_and", "floor_helpers")

    def __init__(self, name: str, floordiv: str, mod: str = "%", and_op: str = "and",
                 select_style: str = "python", isqrt_name: str = "isqrt",
                 arange: Optional[str] = None, paren_cmp_in_and: bool = False,
                 floor_helpers: Optional[tuple] = None):
        for k, v in locals().items():
            if k != "self":
                object.__setattr__(self, k, v)

    def __setattr__(self, k, v):
        raise AttributeError("TargetProfile is immutable")

    def _key(self):
        return tuple(getattr(self, k) for k in self.__slots__)

    def __eq__(self, other):
        return isinstance(other, TargetProfile) and other._key() == self._key()

    def __hash__(self):
        return hash(self._key())

    def __repr__(self):
        return f"TargetProfile(name={self.name!r})"


C_PROFILE = TargetProfile("c", floordiv="/", and_op="&&", select_style="c")
PYTHON_PROFILE = TargetProfile("python", floordiv="//")
TRITON_PROFILE = TargetProfile("triton", floordiv="//", and_op="&", select_style="where",
                               arange="tl.arange", paren_cmp_in_and=True)
CUDA_PROFILE = TargetProfile("cuda", floordiv="/", and_op="&&", select_style="c",
                             isqrt_name="lego_isqrt", floor_helpers=("lego_fdiv", "lego_fmod"))

PROFILES = {p.name: p for p in (C_PROFILE, PYTHON_PROFILE, TRITON_PROFILE, CUDA_PROFILE)}


def get_profile(name: str) -> TargetProfile:
    prof = PROFILES.get(name)
    if prof is None:
        raise UnsupportedNode(f"unknown target profile {name!r}")
    return prof


class RangeExpr:
    """A compile-time constant index range bound to a variable name."""

    __slots__ = ("name", "lo", "hi")

    def __init__(self, name: str, lo: int, hi: int):
        if not (isinstance(lo, int) and isinstance(hi, int)):
            raise UnsupportedNode("range bounds must be integer constants")
        if lo >= hi:
            raise UnsupportedNode(f"empty range [{lo}, {hi})")
        object.__setattr__(self, "name", name)
        object.__setattr__(self, "lo", lo)
        object.__setattr__(self, "hi", hi)

    def __setattr__(self, k, v):
        raise AttributeError("RangeExpr is immutable")

    def __eq__(self, other):
        return isinstance(other, RangeExpr) and (self.name, self.lo, self.hi) == (
            other.name, other.lo, other.hi)

    def __hash__(self):
        return hash((self.name, self.lo, self.hi))

    def __repr__(self):
        return f"RangeExpr(name={self.name!r}, lo={self.lo}, hi={self.hi})"


def emit_range(r: RangeExpr, profile: TargetProfile) -> str:
    if profile.arange is None:
        raise UnsupportedNode(f"profile {profile.name!r} has no range-expression syntax")
    return f"{profile.arange}({r.lo}, {r.hi})"


def broadcast_suffix(axis: int, total: int) -> str:
    if total <= 1:
        return ""
    slots = ["None"] * total
    slots[axis] = ":"
    return "[" + ", ".join(slots) + "]"


# precedence ladder: conditional < additive < multiplicative < atom
P_SEL, P_ADD, P_MUL, P_ATOM = 0, 10, 20, 100


def emit_expr(e: Expr, profile: TargetProfile, *,
              ranges: Optional[Mapping[str, RangeExpr]] = None,
              broadcasts: Optional[Mapping[str, tuple]] = None) -> str:
    if ranges and profile.arange is None:
        raise UnsupportedNode(
            f"range-expression variables are not supported by profile {profile.name!r}")
    return _Printer(profile, ranges or {}, broadcasts or {}).text(e, P_SEL)


class _Printer:
    def __init__(self, profile: TargetProfile, ranges, broadcasts):
        self.p = profile
        self.ranges = ranges
        self.bcast = broadcasts
        self._iv = None

    def nonneg(self, e) -> bool:
        if self._iv is None:
            from .simplify import Intervals
            self._iv = Intervals()
        r = self._iv.maybe(e)
        return r is not None and r[0] >= 0

    def text(self, e, outer: int) -> str:
        t = type(e)
        if t is IntConst:
            s = str(e.value)
            return f"({s})" if e.value < 0 and outer >= P_MUL else s
        if t is Var:
            return self.var(e)
        if t is Add:
            return self.infix(e.lhs, " + ", e.rhs, P_ADD, outer, type(e.rhs) in (Add, Sub))
        if t is Sub:
            return self.infix(e.lhs, " - ", e.rhs, P_ADD, outer, False)
        if t is Mul:
            return self.infix(e.lhs, "*", e.rhs, P_MUL, outer, type(e.rhs) is Mul)
        if t is FloorDiv or t is Mod:
            helpers = self.p.floor_helpers
            if helpers and not (self.nonneg(e.num) and self.nonneg(e.den)):
                fn = helpers[0] if t is FloorDiv else helpers[1]
                return f"{fn}({self.text(e.num, P_SEL)}, {self.text(e.den, P_SEL)})"
            op = f" {self.p.floordiv} " if t is FloorDiv else f" {self.p.mod} "
            return self.infix(e.num, op, e.den, P_MUL, outer, False)
        if t is Select:
            return self.select(e, outer)
        if t is Call:
            fn = self.p.isqrt_name if e.intrinsic == "isqrt" else e.intrinsic
            return f"{fn}(" + ", ".join(self.text(a, P_SEL) for a in e.args) + ")"
        raise UnsupportedNode(f"cannot emit {type(e).__name__}")

    def var(self, v: Var) -> str:
        r = self.ranges.get(v.name)
        s = emit_range(r, self.p) if r is not None else v.name
        b = self.bcast.get(v.name)
        if b is not None:
            suffix = broadcast_suffix(*b)
            if suffix:
                return f"({s}){suffix}"
        return s

    def infix(self, lhs, op, rhs, prec, outer, assoc_rhs):
        # left-associative operators: an equal-precedence right operand needs
        # parentheses unless the chain is associative (a + (b - c), a*(b*c))
        s = self.text(lhs, prec - 1) + op + self.text(rhs, prec - 1 if assoc_rhs else prec)
        return f"({s})" if prec <= outer else s

    def select(self, e: Select, outer: int) -> str:
        c = self.cond(e.cond)
        a, b = self.text(e.then, P_SEL), self.text(e.orelse, P_SEL)
        style = self.p.select_style
        if style == "where":
            return f"tl.where({c}, {a}, {b})"
        s = f"{c} ? {a} : {b}" if style == "c" else f"{a} if {c} else {b}"
        return f"({s})" if outer > P_SEL else s

    def cond(self, c) -> str:
        if type(c) is Cmp:
            return f"{self.text(c.lhs, P_ADD - 1)} {c.op} {self.text(c.rhs, P_ADD - 1)}"
        if type(c) is And:
            parts = []
            for side in (c.lhs, c.rhs):
                s = self.cond(side)
                if self.p.paren_cmp_in_and and type(side) is Cmp:
                    s = f"({s})"
                parts.append(s)
            return f" {self.p.and_op} ".join(parts)
        raise UnsupportedNode(f"cannot emit condition {type(c).__name__}")
