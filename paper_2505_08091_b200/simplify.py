"""Range analysis and algebraic simplification of index expressions.

Public surface mirrors the reference (``pkg/src/lego/simplify.py``):
``FactSet`` (``:38-79``), ``range_of`` (``:86``), ``simplify`` (``:626``) and
``best_variant`` (``:635-644``).  The *engine* is different.  The reference
rewrites trees innermost-first with seven Table-II div/mod rules under a
firing budget; this module normalises bottom-up into linear forms
(``{atom: coefficient} + constant``) over which the same identities become
direct operations:

* ``(d*q + r) // d -> q + r // d`` and ``(d*q + r) % d -> r % d`` (Table II
  rules 1-2), with the constant of ``r`` reduced into ``[0, d)``;
* ``x // a -> 0`` / ``x % a -> x`` when ``0 <= x < a`` (rules 4-5) and the
  ``(x % d) // d -> 0`` special case (rule 3);
* ``a*(x // a) + x % a -> x`` (rule 7, recomposition) generalised to digit
  merging ``a*((x // a) % b) + x % a -> x % (a*b)``;
* nested constant divisors ``(x // a) // b -> x // (a*b)`` and
  ``(x % (a*b)) // a -> (x // a) % b``, which the reference leaves unmerged
   -- the CUDA code generator wants them merged.

Every identity used holds for *all* integers under floor semantics, so the
rewrite is sound without sign proofs except where a range test is stated.
"""

from __future__ import annotations

import math
import threading
from typing import Dict, Iterable, Mapping, Optional, Tuple

from .errors import DivisionByZero, UnboundVariable
from .expr import (
    Add,
    And,
    Call,
    Cmp,
    Cond,
    Expr,
    FloorDiv,
    IntConst,
    Mod,
    Mul,
    Select,
    Sub,
    Var,
    VarRange,
    expand,
    op_count,
)

DEFAULT_BUDGET = 10_000


class FactSet:
    """Variable ranges plus divisibility facts ``var % k == 0`` (k >= 2)."""

    __slots__ = ("ranges", "divisibility")

    def __init__(self, ranges: Optional[Mapping[str, VarRange]] = None,
                 divisibility: Iterable[Tuple[str, int]] = ()):
        self.ranges = dict(ranges or {})
        self.divisibility = frozenset(divisibility)
        bad = [k for _, k in self.divisibility if k < 2]
        if bad:
            raise ValueError(f"divisibility modulus must be >= 2, got {bad[0]}")

    def with_range(self, name: str, rng: VarRange) -> "FactSet":
        r = dict(self.ranges)
        r[name] = rng
        return FactSet(r, self.divisibility)

    def with_divisibility(self, name: str, k: int) -> "FactSet":
        return FactSet(self.ranges, self.divisibility | {(name, k)})

    def merged(self, other: "FactSet") -> "FactSet":
        r = dict(self.ranges)
        for name, rng in other.ranges.items():
            r[name] = r[name].intersect(rng) if name in r else rng
        return FactSet(r, self.divisibility | other.divisibility)

    def range_for(self, name: str) -> Optional[VarRange]:
        return self.ranges.get(name)

    def divisors_of(self, name: str):
        return {k for n, k in self.divisibility if n == name}

    def __repr__(self):
        items = [f"{n} in {r}" for n, r in sorted(self.ranges.items())]
        items += [f"{n} % {k} == 0" for n, k in sorted(self.divisibility)]
        return "FactSet(" + ", ".join(items) + ")"


EMPTY_FACTS = FactSet()


# ---------------------------------------------------------------------------
# Interval analysis (closed intervals internally).
# ---------------------------------------------------------------------------

def range_of(e: Expr, facts: FactSet = EMPTY_FACTS) -> VarRange:
    """Sound half-open over-approximation of the values ``e`` can take."""
    lo, hi = Intervals(facts).of(e)
    return VarRange(lo, hi + 1)


class Intervals:
    """Memoised interval evaluator; raises UnboundVariable for unranged vars."""

    def __init__(self, facts: FactSet = EMPTY_FACTS):
        self.facts = facts
        self.memo: Dict[Expr, Tuple[int, int]] = {}

    def of(self, e) -> Tuple[int, int]:
        got = self.memo.get(e)
        if got is None:
            got = self._raw(e)
            self.memo[e] = got
        return got

    def maybe(self, e) -> Optional[Tuple[int, int]]:
        try:
            return self.of(e)
        except (UnboundVariable, DivisionByZero, ValueError):
            return None

    def _raw(self, e):
        t = type(e)
        if t is IntConst:
            return (e.value, e.value)
        if t is Var:
            rng = e.range
            fr = self.facts.range_for(e.name)
            if fr is not None:
                rng = fr if rng is None else fr.intersect(rng)
            if rng is None:
                raise UnboundVariable(e.name)
            return (rng.lo, rng.hi - 1)
        if t is Add:
            a, b = self.of(e.lhs), self.of(e.rhs)
            return (a[0] + b[0], a[1] + b[1])
        if t is Sub:
            a, b = self.of(e.lhs), self.of(e.rhs)
            return (a[0] - b[1], a[1] - b[0])
        if t is Mul:
            a, b = self.of(e.lhs), self.of(e.rhs)
            p = (a[0] * b[0], a[0] * b[1], a[1] * b[0], a[1] * b[1])
            return (min(p), max(p))
        if t is FloorDiv:
            return _iv_div(self.of(e.num), self.of(e.den))
        if t is Mod:
            return _iv_mod(self.of(e.num), self.of(e.den))
        if t is Select:
            a, b = self.of(e.then), self.of(e.orelse)
            return (min(a[0], b[0]), max(a[1], b[1]))
        if t is Call:
            a = self.of(e.args[0])
            return (math.isqrt(max(a[0], 0)), math.isqrt(max(a[1], 0)))
        raise TypeError(f"not an expression: {e!r}")

    def decide(self, c: Cond) -> Optional[bool]:
        """True / False when the condition is constant over all ranges."""
        if type(c) is And:
            a, b = self.decide(c.lhs), self.decide(c.rhs)
            if a is False or b is False:
                return False
            return True if (a is True and b is True) else None
        ra, rb = self.maybe(c.lhs), self.maybe(c.rhs)
        if ra is None or rb is None:
            return None
        (alo, ahi), (blo, bhi) = ra, rb
        op = c.op
        if op == "<":
            return True if ahi < blo else (False if alo >= bhi else None)
        if op == "<=":
            return True if ahi <= blo else (False if alo > bhi else None)
        if op == ">":
            return True if alo > bhi else (False if ahi <= blo else None)
        if op == ">=":
            return True if alo >= bhi else (False if ahi < blo else None)
        if alo == ahi == blo == bhi:
            return True
        return False if (ahi < blo or alo > bhi) else None


def _split_den(den):
    lo, hi = den
    if lo == 0 and hi == 0:
        raise DivisionByZero("divisor interval is exactly zero")
    parts = []
    if lo < 0:
        parts.append((lo, min(hi, -1)))
    if hi > 0:
        parts.append((max(lo, 1), hi))
    return parts


def _iv_div(num, den):
    vals = [n // d for lo_hi in _split_den(den) for n in num for d in lo_hi]
    return (min(vals), max(vals))


def _iv_mod(num, den):
    nlo, nhi = num
    lo, hi = [], []
    for dlo, dhi in _split_den(den):
        if dlo > 0:
            if nlo >= 0 and nhi < dlo:
                lo.append(nlo)
                hi.append(nhi)
            else:
                lo.append(0)
                hi.append(min(dhi - 1, nhi) if nlo >= 0 else dhi - 1)
        else:
            lo.append(dlo + 1)
            hi.append(0)
    return (min(lo), max(hi))


# ---------------------------------------------------------------------------
# Linear forms.
# ---------------------------------------------------------------------------

class Lin:
    """``sum(coef * atom) + const``; atoms keep first-insertion order."""

    __slots__ = ("terms", "const")

    def __init__(self, terms=None, const=0):
        self.terms: Dict[Expr, int] = terms if terms is not None else {}
        self.const = const

    def copy(self):
        return Lin(dict(self.terms), self.const)

    def add(self, other: "Lin", sign=1):
        for a, c in other.terms.items():
            v = self.terms.get(a, 0) + sign * c
            if v:
                self.terms[a] = v
            else:
                self.terms.pop(a, None)
        self.const += sign * other.const
        return self

    def scaled(self, k: int) -> "Lin":
        if k == 0:
            return Lin()
        return Lin({a: c * k for a, c in self.terms.items()}, self.const * k)

    def is_const(self):
        return not self.terms


def _lin_of(e: Expr) -> Lin:
    """Linear view of an already-normalised expression."""
    t = type(e)
    if t is IntConst:
        return Lin({}, e.value)
    if t is Add or t is Sub:
        out = _lin_of(e.lhs).copy()
        return out.add(_lin_of(e.rhs), 1 if t is Add else -1)
    if t is Mul:
        if type(e.rhs) is IntConst:
            return _lin_of(e.lhs).scaled(e.rhs.value)
        if type(e.lhs) is IntConst:
            return _lin_of(e.rhs).scaled(e.lhs.value)
    return Lin({e: 1}, 0)


def _term(atom: Expr, mag: int) -> Expr:
    if mag == 1:
        return atom
    # expanded variants print coefficient-first (2*i, like expand()); plain
    # ones keep the stride form that canonical flattening produces (i*8)
    return Mul(atom, IntConst(mag)) if getattr(_MODE, "factor", True) else Mul(IntConst(mag), atom)


_MODE = threading.local()     # factor_gcd switch of the running simplify() call


def _build(lin: Lin) -> Expr:
    if len(lin.terms) > 1 and getattr(_MODE, "factor", True):
        g = math.gcd(lin.const, *lin.terms.values())
        if g > 1:
            # keep a common factor factored out: 2*(i + j), not i*2 + j*2
            inner = Lin({a: c // g for a, c in lin.terms.items()}, lin.const // g)
            return Mul(IntConst(g), _build(inner))
    pos = [(a, c) for a, c in lin.terms.items() if c > 0]
    neg = [(a, -c) for a, c in lin.terms.items() if c < 0]
    acc: Optional[Expr] = None
    for a, c in pos:
        acc = _term(a, c) if acc is None else Add(acc, _term(a, c))
    if acc is None:
        if not neg:
            return IntConst(lin.const)
        if lin.const > 0:
            acc = IntConst(lin.const)
        else:
            acc = IntConst(0) if lin.const == 0 else IntConst(lin.const)
        for a, c in neg:
            acc = Sub(acc, _term(a, c))
        return acc
    for a, c in neg:
        acc = Sub(acc, _term(a, c))
    if lin.const > 0:
        acc = Add(acc, IntConst(lin.const))
    elif lin.const < 0:
        acc = Sub(acc, IntConst(-lin.const))
    return acc


# ---------------------------------------------------------------------------
# The normaliser.
# ---------------------------------------------------------------------------

class _Normaliser:
    def __init__(self, facts: FactSet):
        self.facts = facts
        self.iv = Intervals(facts)
        self.memo: Dict[Expr, Expr] = {}

    # -- helpers ------------------------------------------------------------
    def lin_interval(self, lin: Lin) -> Optional[Tuple[int, int]]:
        lo = hi = lin.const
        for a, c in lin.terms.items():
            r = self.iv.maybe(a)
            if r is None:
                return None
            if c >= 0:
                lo += c * r[0]
                hi += c * r[1]
            else:
                lo += c * r[1]
                hi += c * r[0]
        return (lo, hi)

    def divisible(self, atom: Expr, coef: int, d: int) -> Optional[Expr]:
        """coef*atom / d as an expression when it is an exact multiple."""
        if coef % d == 0:
            return _term_signed(atom, coef // d)
        if type(atom) is Var:
            for k in self.facts.divisors_of(atom.name):
                if (coef * k) % d == 0:
                    return _term_signed(FloorDiv(atom, IntConst(k)), coef * k // d)
        return None

    # -- entry --------------------------------------------------------------
    def run(self, e: Expr) -> Expr:
        got = self.memo.get(e)
        if got is None:
            got = self._norm(e)
            self.memo[e] = got
            self.memo.setdefault(got, got)
        return got

    def _norm(self, e: Expr) -> Expr:
        t = type(e)
        if t is IntConst:
            return e
        if t is Var:
            r = self.iv.maybe(e)
            # a variable pinned to one value by its range is that constant
            return IntConst(r[0]) if r is not None and r[0] == r[1] else e
        if t is Add or t is Sub:
            lin = _lin_of(self.run(e.lhs)).copy()
            lin.add(_lin_of(self.run(e.rhs)), 1 if t is Add else -1)
            return self.finish_sum(lin)
        if t is Mul:
            a, b = self.run(e.lhs), self.run(e.rhs)
            if type(b) is IntConst:
                return self.finish_sum(_lin_of(a).scaled(b.value))
            if type(a) is IntConst:
                return self.finish_sum(_lin_of(b).scaled(a.value))
            return Mul(a, b)
        if t is FloorDiv or t is Mod:
            num, den = self.run(e.num), self.run(e.den)
            if type(den) is IntConst and den.value > 0:
                return self.div_mod(t is FloorDiv, num, den.value)
            if type(num) is IntConst and type(den) is IntConst:
                return IntConst(num.value // den.value if t is FloorDiv else num.value % den.value)
            return t(num, den)
        if t is Select:
            cond = self.cond(e.cond)
            if cond is True:
                return self.run(e.then)
            if cond is False:
                return self.run(e.orelse)
            then, orelse = self.run(e.then), self.run(e.orelse)
            if then == orelse:
                return then
            return Select(cond, then, orelse)
        if t is Call:
            arg = self.run(e.args[0])
            if type(arg) is IntConst and arg.value >= 0:
                return IntConst(math.isqrt(arg.value))
            r = self.iv.maybe(arg)
            if r is not None and r[0] >= 0 and math.isqrt(r[0]) == math.isqrt(r[1]):
                return IntConst(math.isqrt(r[0]))
            return Call(e.intrinsic, (arg,))
        raise TypeError(f"not an expression: {e!r}")

    def cond(self, c: Cond):
        if type(c) is Cmp:
            c2 = Cmp(c.op, self.run(c.lhs), self.run(c.rhs))
            d = self.iv.decide(c2)
            return c2 if d is None else d
        a, b = self.cond(c.lhs), self.cond(c.rhs)
        if a is False or b is False:
            return False
        if a is True:
            return b
        if b is True:
            return a
        return And(a, b)

    # -- sums ---------------------------------------------------------------
    def finish_sum(self, lin: Lin) -> Expr:
        changed = True
        while changed and len(lin.terms) > 1:
            changed = self.merge_digits(lin) or self.fuse_selects(lin)
        return _build(lin)

    def fuse_selects(self, lin: Lin) -> bool:
        """c1*sel(p, a1, b1) + c2*sel(p, a2, b2) -> sel(p, c1*a1 + c2*a2, c1*b1 + c2*b2)."""
        by_cond: Dict = {}
        for atom in lin.terms:
            if type(atom) is Select:
                by_cond.setdefault(atom.cond, []).append(atom)
        for cond, atoms in by_cond.items():
            if len(atoms) < 2:
                continue
            then, orelse = Lin(), Lin()
            for a in atoms:
                c = lin.terms.pop(a)
                then.add(_lin_of(a.then).scaled(c))
                orelse.add(_lin_of(a.orelse).scaled(c))
            fused = self.run(Select(cond, _build(then), _build(orelse)))
            lin.add(_lin_of(fused))
            return True
        return False

    def merge_digits(self, lin: Lin) -> bool:
        """Fold two div/mod atoms over the same base into one atom.

        An atom ``(x // lo) % span`` holds the digits ``[lo, lo*span)`` of x.
        If a second atom holds the digits directly above (``lo2 == lo*span``)
        and carries ``span`` times the first one's coefficient, the pair is the
        single digit run ``(x // lo) % (span*span2)`` (``x // lo`` when the
        upper run is unbounded; plain ``x`` when also ``lo == 1``): this covers
        recomposition ``a*(x // a) + x % a -> x`` and digit merging.  Exact for
        every integer x.
        """
        items = list(lin.terms.items())
        for atom, c in items:
            base, lo, span = _digit_of(atom)
            if base is None or span is None:
                continue
            for other, c2 in items:
                if other is atom:
                    continue
                base2, lo2, span2 = _digit_of(other)
                if base2 is None or lo2 != lo * span or c2 != c * span or base2 != base:
                    continue
                del lin.terms[atom]
                del lin.terms[other]
                merged = self.run(_digit_atom(base, lo, None if span2 is None else span * span2))
                lin.add(_lin_of(merged).scaled(c))
                return True
        return False

    # -- div / mod by a positive constant -----------------------------------
    def div_mod(self, is_div: bool, num: Expr, d: int) -> Expr:
        if d == 1:
            return num if is_div else IntConst(0)
        lin = _lin_of(num)
        quot = Lin()
        rest = Lin({}, 0)
        for a, c in lin.terms.items():
            q = self.divisible(a, c, d)
            if q is None:
                rest.terms[a] = c
            else:
                quot.add(_lin_of(q))
        q0, r0 = divmod(lin.const, d)
        rest.const = r0
        quot.const += q0
        g = math.gcd(d, rest.const, *rest.terms.values())
        if g > 1:
            # (g*Y) // (g*k) == Y // k  and  (g*Y) % (g*k) == g*(Y % k)
            inner = Lin({a: c // g for a, c in rest.terms.items()}, rest.const // g)
            if is_div:
                return self.finish_sum(quot.add(_lin_of(self.div_rest(inner, d // g))))
            return self.finish_sum(_lin_of(self.mod_rest(inner, d // g)).scaled(g))
        if not is_div:
            return self.mod_rest(rest, d)
        return self.finish_sum(quot.add(_lin_of(self.div_rest(rest, d))))

    def split_small(self, rest: Lin, d: int):
        """Find a | d with rest = a*Q + R where every term of Q has a
        coefficient divisible by a and 0 <= R < a.  Then (floor semantics,
        any sign of Q):  rest // d == Q // (d/a)  and
        rest % d == a*(Q % (d/a)) + R.  Returns (a, Q, R) or None."""
        cands = sorted({math.gcd(d, c) for c in rest.terms.values()} - {1, d}, reverse=True)
        for a in cands:
            big = Lin({t: c // a for t, c in rest.terms.items() if c % a == 0}, 0)
            small = Lin({t: c for t, c in rest.terms.items() if c % a != 0}, rest.const)
            if not big.terms:
                continue
            r = self.lin_interval(small)
            if r is not None and r[0] >= 0 and r[1] < a:
                return a, big, small
        return None

    def div_rest(self, rest: Lin, d: int) -> Expr:
        if d == 1:
            return _build(rest)
        r = self.lin_interval(rest)
        if r is not None and r[0] // d == r[1] // d:
            return IntConst(r[0] // d)
        if rest.is_const():
            return IntConst(rest.const // d)
        sp = self.split_small(rest, d)
        if sp is not None:
            a, big, _ = sp
            return self.div_mod(True, _build(big), d // a)
        if len(rest.terms) == 1 and rest.const == 0:
            (a, c), = rest.terms.items()
            if c == 1:
                t = type(a)
                if t is FloorDiv and type(a.den) is IntConst and a.den.value > 0:
                    return self.div_mod(True, a.num, a.den.value * d)
                if t is Mod and type(a.den) is IntConst and a.den.value > 0 and a.den.value % d == 0:
                    # (x % (d*b)) // d -> (x // d) % b
                    inner = self.div_mod(True, a.num, d)
                    return self.div_mod(False, inner, a.den.value // d)
        return FloorDiv(_build(rest), IntConst(d))

    def mod_rest(self, rest: Lin, d: int) -> Expr:
        if d == 1:
            return IntConst(0)
        r = self.lin_interval(rest)
        if r is not None and 0 <= r[0] and r[1] < d:
            return _build(rest)
        if rest.is_const():
            return IntConst(rest.const % d)
        sp = self.split_small(rest, d)
        if sp is not None:
            a, big, small = sp
            hi = _lin_of(self.div_mod(False, _build(big), d // a)).scaled(a)
            return self.finish_sum(hi.add(small))
        if len(rest.terms) == 1 and rest.const == 0:
            (a, c), = rest.terms.items()
            if c == 1 and type(a) is Mod and type(a.den) is IntConst:
                m = a.den.value
                if m > 0 and m % d == 0:
                    return self.div_mod(False, a.num, d)
            if type(a) is Var and any(k % d == 0 for k in self.facts.divisors_of(a.name)):
                return IntConst(0)
        return Mod(_build(rest), IntConst(d))


def _term_signed(atom: Expr, coef: int) -> Expr:
    if coef == 0:
        return IntConst(0)
    if coef == 1:
        return atom
    return Mul(atom, IntConst(coef))


def _digit_of(atom: Expr):
    """View an atom as a run of mixed-radix digits of a base expression.

    Returns (base, lo, span): the atom equals ``(base // lo) % span`` (span
    None means unbounded, i.e. plain ``base // lo``).  Plain non-div atoms
    are ``(atom, 1, None)``.
    """
    t = type(atom)
    if t is FloorDiv and type(atom.den) is IntConst and atom.den.value > 0:
        return atom.num, atom.den.value, None
    if t is Mod and type(atom.den) is IntConst and atom.den.value > 0:
        inner = atom.num
        if type(inner) is FloorDiv and type(inner.den) is IntConst and inner.den.value > 0:
            return inner.num, inner.den.value, atom.den.value
        return inner, 1, atom.den.value
    if t in (IntConst,):
        return None, 0, None
    return atom, 1, None


def _digit_atom(base: Expr, lo: int, span: Optional[int]) -> Expr:
    x = base if lo == 1 else FloorDiv(base, IntConst(lo))
    return x if span is None else Mod(x, IntConst(span))


# ---------------------------------------------------------------------------
# Public entry points.
# ---------------------------------------------------------------------------

def simplify(e: Expr, facts: FactSet = EMPTY_FACTS, *, budget: int = DEFAULT_BUDGET,
             factor_gcd: bool = True) -> Expr:
    """Semantically equal, usually smaller expression; never raises.

    ``budget`` bounds the number of whole-expression normalisation passes
    (each pass is linear in the DAG size); it exists for API parity with the
    reference, whose budget counts individual rule firings.  ``factor_gcd``
    keeps a common constant factor of a sum factored out (``2*(i + j)``);
    the expanded variants switch it off so they stay fully distributed.
    """
    if budget <= 0:
        return e
    passes = min(budget, 8)
    cur = e
    prev = getattr(_MODE, "factor", True)
    _MODE.factor = factor_gcd
    try:
        for _ in range(passes):
            try:
                nxt = _Normaliser(facts).run(cur)
            except (UnboundVariable, DivisionByZero, ValueError):
                return cur
            if nxt == cur:
                return nxt
            cur = nxt
        return cur
    finally:
        _MODE.factor = prev


def best_variant(e: Expr, facts: FactSet = EMPTY_FACTS, *, budget: int = DEFAULT_BUDGET) -> Expr:
    """Cheaper (by ``op_count``) of ``simplify(e)`` and ``simplify(expand(e))``;
    ties keep the unexpanded form (reference ``simplify.py:635-644``)."""
    plain = simplify(e, facts, budget=budget)
    alt = simplify(expand(e), facts, budget=budget, factor_gcd=False)
    return alt if op_count(alt) < op_count(plain) else plain


# The paper's Table-II rules one by one, under the reference's names (its
# tests import them from here); this engine subsumes them (see rules.py).
from .rules import (  # noqa: E402,F401
    TABLE_RULES,
    _Prover,
    rule_div_below_bound,
    rule_div_by_one_assoc,
    rule_div_of_mod,
    rule_div_of_multiple_sum,
    rule_mod_below_bound,
    rule_mod_of_multiple_sum,
    rule_recompose,
)
