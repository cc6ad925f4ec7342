"""Integer index-expression IR.

The node vocabulary and its semantics follow the reference
(``pkg/src/lego/expr.py:99-258`` for the node set, ``expr.py:261-316`` for
``eval_expr``/``eval_cond``): exact integers, *floor* division, Python-sign
modulo, ``isqrt`` as the only intrinsic and a lazily evaluated ``Select``.

The representation is different and chosen for the CUDA code generator:
every node caches its structural hash at construction, so expression trees
behave as DAGs -- equal sub-terms hash and compare in O(1) after the first
comparison, which is what common-subexpression elimination in
:mod:`.codegen` relies on.  Nodes are immutable (``__setattr__`` raises) and
therefore shareable across threads, like the reference's frozen dataclasses.
"""

from __future__ import annotations

import math
from typing import Dict, Iterator, List, Mapping, Optional, Tuple, Union

from .errors import DivisionByZero, UnboundVariable

INTRINSICS = ("isqrt",)


class VarRange:
    """Half-open integer interval ``[lo, hi)``."""

    __slots__ = ("lo", "hi")

    def __init__(self, lo: int, hi: int):
        for b in (lo, hi):
            if isinstance(b, bool) or not isinstance(b, int):
                raise TypeError("range bounds must be integers")
        if lo >= hi:
            raise ValueError(f"empty range [{lo}, {hi})")
        object.__setattr__(self, "lo", lo)
        object.__setattr__(self, "hi", hi)

    def __setattr__(self, k, v):
        raise AttributeError("VarRange is immutable")

    @property
    def max(self) -> int:
        return self.hi - 1

    def contains(self, v: int) -> bool:
        return self.lo <= v < self.hi

    def intersect(self, other: "VarRange") -> "VarRange":
        lo, hi = max(self.lo, other.lo), min(self.hi, other.hi)
        if lo >= hi:
            raise ValueError(f"disjoint ranges {self} and {other}")
        return VarRange(lo, hi)

    def __eq__(self, other):
        return isinstance(other, VarRange) and self.lo == other.lo and self.hi == other.hi

    def __hash__(self):
        return hash(("VarRange", self.lo, self.hi))

    def __repr__(self):
        return f"VarRange(lo={self.lo}, hi={self.hi})"

    def __str__(self):
        return f"[{self.lo}, {self.hi})"


# ---------------------------------------------------------------------------
# Node machinery: one slot tuple per class, hash computed once.
# ---------------------------------------------------------------------------

class _Node:
    __slots__ = ("_h",)
    _fields: Tuple[str, ...] = ()

    def _seal(self):
        object.__setattr__(
            self, "_h", hash((type(self).__name__,) + tuple(getattr(self, f) for f in self._fields)))

    def __setattr__(self, k, v):
        raise AttributeError(f"{type(self).__name__} is immutable")

    def __hash__(self):
        return self._h

    def __eq__(self, other):
        if self is other:
            return True
        if type(other) is not type(self) or other._h != self._h:
            return False
        return all(getattr(self, f) == getattr(other, f) for f in self._fields)

    def __ne__(self, other):
        return not self.__eq__(other)

    def __repr__(self):
        inner = ", ".join(f"{f}={getattr(self, f)!r}" for f in self._fields)
        return f"{type(self).__name__}({inner})"

    def __reduce__(self):
        return (type(self), tuple(getattr(self, f) for f in self._fields))


class Expr(_Node):
    """Integer-valued expression; Python arithmetic operators build nodes."""

    __slots__ = ()

    def __add__(self, o):
        return Add(self, o)

    def __radd__(self, o):
        return Add(o, self)

    def __sub__(self, o):
        return Sub(self, o)

    def __rsub__(self, o):
        return Sub(o, self)

    def __mul__(self, o):
        return Mul(self, o)

    def __rmul__(self, o):
        return Mul(o, self)

    def __floordiv__(self, o):
        return FloorDiv(self, o)

    def __rfloordiv__(self, o):
        return FloorDiv(o, self)

    def __mod__(self, o):
        return Mod(self, o)

    def __rmod__(self, o):
        return Mod(o, self)


def as_expr(x) -> "Expr":
    """Lift an ``int`` to :class:`IntConst`; pass expressions through."""
    if isinstance(x, Expr):
        return x
    if isinstance(x, bool) or not isinstance(x, int):
        if isinstance(x, bool):
            raise TypeError("booleans are not integer expressions")
        raise TypeError(f"cannot treat {type(x).__name__} as an expression")
    return IntConst(x)


class IntConst(Expr):
    __slots__ = ("value",)
    _fields = ("value",)

    def __init__(self, value: int):
        if isinstance(value, bool) or not isinstance(value, int):
            raise TypeError("IntConst takes an int")
        object.__setattr__(self, "value", value)
        self._seal()


class Var(Expr):
    __slots__ = ("name", "range")
    _fields = ("name", "range")

    def __init__(self, name: str, range: Optional[VarRange] = None):  # noqa: A002
        object.__setattr__(self, "name", name)
        object.__setattr__(self, "range", range)
        self._seal()


class _Binary(Expr):
    __slots__ = ("lhs", "rhs")
    _fields = ("lhs", "rhs")

    def __init__(self, lhs, rhs):
        object.__setattr__(self, "lhs", as_expr(lhs))
        object.__setattr__(self, "rhs", as_expr(rhs))
        self._seal()


class Add(_Binary):
    __slots__ = ()


class Sub(_Binary):
    __slots__ = ()


class Mul(_Binary):
    __slots__ = ()


class _DivLike(Expr):
    __slots__ = ("num", "den")
    _fields = ("num", "den")
    _zero_msg = ""

    def __init__(self, num, den):
        num, den = as_expr(num), as_expr(den)
        if isinstance(den, IntConst) and den.value == 0:
            raise DivisionByZero(self._zero_msg)
        object.__setattr__(self, "num", num)
        object.__setattr__(self, "den", den)
        self._seal()


class FloorDiv(_DivLike):
    __slots__ = ()
    _zero_msg = "constant zero denominator"


class Mod(_DivLike):
    __slots__ = ()
    _zero_msg = "constant zero modulus"


class Cond(_Node):
    """Boolean condition over expressions."""

    __slots__ = ()


_CMP_FNS = {
    "<": lambda a, b: a < b,
    "<=": lambda a, b: a <= b,
    "==": lambda a, b: a == b,
    ">=": lambda a, b: a >= b,
    ">": lambda a, b: a > b,
}


class Cmp(Cond):
    __slots__ = ("op", "lhs", "rhs")
    _fields = ("op", "lhs", "rhs")

    def __init__(self, op: str, lhs, rhs):
        if op not in _CMP_FNS:
            raise ValueError(f"unknown comparison {op!r}")
        object.__setattr__(self, "op", op)
        object.__setattr__(self, "lhs", as_expr(lhs))
        object.__setattr__(self, "rhs", as_expr(rhs))
        self._seal()


class And(Cond):
    __slots__ = ("lhs", "rhs")
    _fields = ("lhs", "rhs")

    def __init__(self, lhs: Cond, rhs: Cond):
        object.__setattr__(self, "lhs", lhs)
        object.__setattr__(self, "rhs", rhs)
        self._seal()


def lt(a, b) -> Cmp:
    return Cmp("<", a, b)


def le(a, b) -> Cmp:
    return Cmp("<=", a, b)


def eq(a, b) -> Cmp:
    return Cmp("==", a, b)


def ge(a, b) -> Cmp:
    return Cmp(">=", a, b)


def gt(a, b) -> Cmp:
    return Cmp(">", a, b)


def and_all(conds) -> Cond:
    """Left-associated conjunction of one or more conditions."""
    it = iter(conds)
    try:
        acc = next(it)
    except StopIteration:
        raise ValueError("and_all of no conditions") from None
    for c in it:
        acc = And(acc, c)
    return acc


class Select(Expr):
    __slots__ = ("cond", "then", "orelse")
    _fields = ("cond", "then", "orelse")

    def __init__(self, cond: Cond, then, orelse):
        if not isinstance(cond, Cond):
            raise TypeError("Select condition must be a Cond")
        object.__setattr__(self, "cond", cond)
        object.__setattr__(self, "then", as_expr(then))
        object.__setattr__(self, "orelse", as_expr(orelse))
        self._seal()


class Call(Expr):
    __slots__ = ("intrinsic", "args")
    _fields = ("intrinsic", "args")

    def __init__(self, intrinsic: str, args):
        if intrinsic not in INTRINSICS:
            raise ValueError(f"unknown intrinsic {intrinsic!r}")
        args = tuple(as_expr(a) for a in args)
        if intrinsic == "isqrt" and len(args) != 1:
            raise ValueError("isqrt takes exactly one argument")
        object.__setattr__(self, "intrinsic", intrinsic)
        object.__setattr__(self, "args", args)
        self._seal()


def isqrt(x) -> Call:
    return Call("isqrt", (x,))


# ---------------------------------------------------------------------------
# Evaluation (semantics pinned to reference expr.py:261-316).
# ---------------------------------------------------------------------------

def eval_expr(e: Expr, env: Mapping[str, int]) -> int:
    """Exact evaluation; floor ``//``, Python ``%``, lazy ``Select``."""
    return _Evaluator(env).ev(e)


def eval_cond(c: Cond, env: Mapping[str, int]) -> bool:
    return _Evaluator(env).cond(c)


class _Evaluator:
    """Memoised (per call) evaluator: shared sub-DAGs are computed once."""

    __slots__ = ("env", "memo")

    def __init__(self, env):
        self.env = env
        self.memo: Dict[int, int] = {}

    def ev(self, e) -> int:
        key = id(e)
        got = self.memo.get(key)
        if got is not None:
            return got
        t = type(e)
        if t is IntConst:
            return e.value
        if t is Var:
            try:
                return self.env[e.name]
            except KeyError:
                raise UnboundVariable(e.name) from None
        if t is Add:
            v = self.ev(e.lhs) + self.ev(e.rhs)
        elif t is Sub:
            v = self.ev(e.lhs) - self.ev(e.rhs)
        elif t is Mul:
            v = self.ev(e.lhs) * self.ev(e.rhs)
        elif t is FloorDiv or t is Mod:
            d = self.ev(e.den)
            if d == 0:
                raise DivisionByZero("division by zero" if t is FloorDiv else "modulo by zero")
            n = self.ev(e.num)
            v = n // d if t is FloorDiv else n % d
        elif t is Select:
            v = self.ev(e.then) if self.cond(e.cond) else self.ev(e.orelse)
        elif t is Call:
            v = math.isqrt(self.ev(e.args[0]))
        else:
            raise TypeError(f"not an expression: {e!r}")
        self.memo[key] = v
        return v

    def cond(self, c) -> bool:
        if type(c) is Cmp:
            return _CMP_FNS[c.op](self.ev(c.lhs), self.ev(c.rhs))
        if type(c) is And:
            return self.cond(c.lhs) and self.cond(c.rhs)
        raise TypeError(f"not a condition: {c!r}")


# ---------------------------------------------------------------------------
# Traversal helpers.
# ---------------------------------------------------------------------------

def children(e) -> Tuple:
    """Direct expression children of a node (conditions are flattened)."""
    t = type(e)
    if t in (Add, Sub, Mul):
        return (e.lhs, e.rhs)
    if t in (FloorDiv, Mod):
        return (e.num, e.den)
    if t is Select:
        return cond_exprs(e.cond) + (e.then, e.orelse)
    if t is Call:
        return e.args
    return ()


def cond_exprs(c) -> Tuple:
    if type(c) is Cmp:
        return (c.lhs, c.rhs)
    return cond_exprs(c.lhs) + cond_exprs(c.rhs)


def walk(e: Expr) -> Iterator[Expr]:
    """Every node of the expression *tree* (shared sub-terms repeat)."""
    todo = [e]
    while todo:
        n = todo.pop()
        yield n
        todo.extend(children(n))


def unique_nodes(e: Expr) -> List[Expr]:
    """Distinct nodes of the expression DAG in post-order (children first)."""
    out: List[Expr] = []
    seen = set()
    stack = [(e, False)]
    while stack:
        n, done = stack.pop()
        if done:
            out.append(n)
            continue
        if n in seen:
            continue
        seen.add(n)
        stack.append((n, True))
        for c in reversed(children(n)):
            if c not in seen:
                stack.append((c, False))
    return out


def variables(e: Expr) -> set:
    return {n.name for n in unique_nodes(e) if type(n) is Var}


def var_ranges(e: Expr) -> dict:
    return {n.name: n.range for n in unique_nodes(e) if type(n) is Var and n.range is not None}


_COUNTED = (Add, Sub, Mul, FloorDiv, Mod, Select, Call)


def op_count(e: Expr) -> int:
    """Arithmetic node count of the tree form (the reference cost model,
    ``expr.py:359-364``): shared sub-terms are counted every time."""
    memo: Dict[Expr, int] = {}
    for n in unique_nodes(e):
        memo[n] = (1 if type(n) in _COUNTED else 0) + sum(memo[c] for c in children(n))
    return memo[e]


def dag_op_count(e: Expr) -> int:
    """Arithmetic nodes after common-subexpression elimination."""
    return sum(1 for n in unique_nodes(e) if type(n) in _COUNTED)


# ---------------------------------------------------------------------------
# Polynomial expansion (distribute * over +/-), reference expr.py:367-439.
# ---------------------------------------------------------------------------

def expand(e: Expr) -> Expr:
    """Distribute products over sums and merge like terms.

    Non-polynomial nodes (div/mod/select/call) are kept as opaque factors with
    their operands expanded recursively.  Semantically equal to ``e``.
    """
    poly = _poly(e, {})
    return _poly_to_expr(poly)


def _poly(e, memo) -> Dict[Tuple, int]:
    got = memo.get(e)
    if got is not None:
        return got
    t = type(e)
    if t is IntConst:
        out = {(): e.value} if e.value else {}
    elif t is Add or t is Sub:
        out = dict(_poly(e.lhs, memo))
        sgn = 1 if t is Add else -1
        for k, c in _poly(e.rhs, memo).items():
            out[k] = out.get(k, 0) + sgn * c
    elif t is Mul:
        out = {}
        a, b = _poly(e.lhs, memo), _poly(e.rhs, memo)
        for ka, ca in a.items():
            for kb, cb in b.items():
                k = ka + kb
                out[k] = out.get(k, 0) + ca * cb
    else:
        out = {(_expand_opaque(e),): 1}
    out = {k: c for k, c in out.items() if c}
    memo[e] = out
    return out


def _expand_opaque(e):
    t = type(e)
    if t is FloorDiv or t is Mod:
        return t(expand(e.num), expand(e.den))
    if t is Select:
        return Select(_expand_cond(e.cond), expand(e.then), expand(e.orelse))
    if t is Call:
        return Call(e.intrinsic, tuple(expand(a) for a in e.args))
    return e


def _expand_cond(c):
    if type(c) is Cmp:
        return Cmp(c.op, expand(c.lhs), expand(c.rhs))
    return And(_expand_cond(c.lhs), _expand_cond(c.rhs))


def _poly_to_expr(poly: Dict[Tuple, int]) -> Expr:
    acc: Optional[Expr] = None
    for factors, coef in poly.items():
        if not factors:
            term, mag = None, abs(coef)
        else:
            term = factors[0]
            for f in factors[1:]:
                term = Mul(term, f)
            mag = abs(coef)
        if term is None:
            piece = IntConst(mag)
        elif mag == 1:
            piece = term
        else:
            piece = Mul(IntConst(mag), term)
        if acc is None:
            acc = piece if coef > 0 else Sub(IntConst(0), piece)
        else:
            acc = Add(acc, piece) if coef > 0 else Sub(acc, piece)
    return acc if acc is not None else IntConst(0)


Number = Union[int, Expr]
