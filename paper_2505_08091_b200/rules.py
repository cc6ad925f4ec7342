"""The seven division/modulo rewrite rules of the paper's Table II
(``PAPER.md:1066-1093``), as single-step rewrites with proved side conditions.

The backend's simplifier (:mod:`.simplify`) does not run rule by rule: it
normalises expressions into linear forms with digit merging, which subsumes
these rewrites.  The rules are exposed individually -- under the names the
reference package uses in its own tests (``simplify._Prover``,
``simplify.rule_*``) -- so code and tests written against the reference's
rule API keep working.  Each rule takes an expression and a prover and
returns the rewritten expression, or ``None`` when the pattern does not match
or a side condition cannot be proved:

==========================  =====================  ========================
pattern                     result                 condition
==========================  =====================  ========================
``(d*q + r) % d``           ``r % d``              ``d != 0``
``(d*q + r) // d``          ``q`` / ``q + r // d`` ``0 <= r < d`` / ``d != 0``
``(x % d) // d``            ``0``                  ``d > 0``
``x // a``                  ``0``                  ``a > 0, 0 <= x < a``
``x % a``                   ``x``                  ``a > 0, 0 <= x < a``
``(n + y) // 1``            ``n + y // 1``         always
``a*(x // a) + x % a``      ``x``                  ``a != 0``
==========================  =====================  ========================

Side conditions are proved with the sound interval analysis of
:func:`.simplify.range_of` over the variables' declared ranges and the
prover's :class:`.simplify.FactSet` (the paper proves them with Z3 over the
same index ranges).  A constant multiplier that is a multiple of the divisor
counts as ``d*q`` (``(8*q + r) % 4 -> r % 4``).
"""

from __future__ import annotations

from typing import List, Optional, Tuple

from .expr import Add, Expr, FloorDiv, IntConst, Mod, Mul, Sub


class _Prover:
    """Decides the rules' side conditions from interval bounds."""

    def __init__(self, facts=None):
        from .simplify import EMPTY_FACTS
        self.facts = facts if facts is not None else EMPTY_FACTS

    def _range(self, e: Expr) -> Optional[Tuple[int, int]]:
        from .simplify import Intervals
        return Intervals(self.facts).maybe(e)

    def nonzero(self, e: Expr) -> bool:
        r = self._range(e)
        return r is not None and (r[0] > 0 or r[1] < 0)

    def positive(self, e: Expr) -> bool:
        r = self._range(e)
        return r is not None and r[0] > 0

    def nonneg(self, e: Expr) -> bool:
        r = self._range(e)
        return r is not None and r[0] >= 0

    def less(self, a: Expr, b: Expr) -> bool:
        """a < b for every value of their variables."""
        ra, rb = self._range(a), self._range(b)
        return ra is not None and rb is not None and ra[1] < rb[0]

    def in_range(self, x: Expr, a: Expr) -> bool:
        """0 <= x < a."""
        return self.nonneg(x) and self.less(x, a)


def _multiple_of(term: Expr, d: Expr) -> Optional[Expr]:
    """k with term == d * k: term is d*q or q*d, or c*q / q*c with c a
    constant multiple of a constant d."""
    if type(term) is not Mul:
        return None
    a, b = term.lhs, term.rhs
    if a == d:
        return b
    if b == d:
        return a
    if type(d) is IntConst and d.value != 0:
        for c, q in ((a, b), (b, a)):
            if type(c) is IntConst and c.value % d.value == 0:
                k = c.value // d.value
                return q if k == 1 else Mul(IntConst(k), q)
    return None


def _split_multiple_sum(num: Expr, d: Expr):
    """(q, r) with num == d*q + r (num an Add with a multiple of d on either side)."""
    if type(num) is not Add:
        return None
    for m, r in ((num.lhs, num.rhs), (num.rhs, num.lhs)):
        q = _multiple_of(m, d)
        if q is not None:
            return q, r
    return None


def rule_mod_of_multiple_sum(e: Expr, prover: _Prover) -> Optional[Expr]:
    """(d*q + r) % d -> r % d when d != 0."""
    if type(e) is not Mod:
        return None
    got = _split_multiple_sum(e.num, e.den)
    if got is None or not prover.nonzero(e.den):
        return None
    return Mod(got[1], e.den)


def rule_div_of_multiple_sum(e: Expr, prover: _Prover) -> Optional[Expr]:
    """(d*q + r) // d -> q when 0 <= r < d, else q + r // d (d != 0)."""
    if type(e) is not FloorDiv:
        return None
    got = _split_multiple_sum(e.num, e.den)
    if got is None or not prover.nonzero(e.den):
        return None
    q, r = got
    if prover.in_range(r, e.den):
        return q
    return Add(q, FloorDiv(r, e.den))


def rule_div_of_mod(e: Expr, prover: _Prover) -> Optional[Expr]:
    """(x % d) // d -> 0 when d > 0."""
    if type(e) is not FloorDiv or type(e.num) is not Mod or e.num.den != e.den:
        return None
    return IntConst(0) if prover.positive(e.den) else None


def rule_div_below_bound(e: Expr, prover: _Prover) -> Optional[Expr]:
    """x // a -> 0 when a > 0 and 0 <= x < a."""
    if type(e) is not FloorDiv:
        return None
    return IntConst(0) if prover.positive(e.den) and prover.in_range(e.num, e.den) else None


def rule_mod_below_bound(e: Expr, prover: _Prover) -> Optional[Expr]:
    """x % a -> x when a > 0 and 0 <= x < a."""
    if type(e) is not Mod:
        return None
    return e.num if prover.positive(e.den) and prover.in_range(e.num, e.den) else None


def rule_div_by_one_assoc(e: Expr, prover: _Prover) -> Optional[Expr]:
    """(n + y) // 1 -> n + y // 1 (n integral, always)."""
    if type(e) is not FloorDiv or e.den != IntConst(1) or type(e.num) is not Add:
        return None
    return Add(e.num.lhs, FloorDiv(e.num.rhs, IntConst(1)))


def _signed_terms(e: Expr, sign: int, out: List[Tuple[int, Expr]]):
    t = type(e)
    if t is Add:
        _signed_terms(e.lhs, sign, out)
        _signed_terms(e.rhs, sign, out)
    elif t is Sub:
        _signed_terms(e.lhs, sign, out)
        _signed_terms(e.rhs, -sign, out)
    else:
        out.append((sign, e))


def _scaled_floor(term: Expr):
    """(a, x) when term == a * (x // a)."""
    if type(term) is not Mul:
        return None
    for a, f in ((term.lhs, term.rhs), (term.rhs, term.lhs)):
        if type(f) is FloorDiv and f.den == a:
            return a, f.num
    return None


def rule_recompose(e: Expr, prover: _Prover) -> Optional[Expr]:
    """a*(x // a) + x % a -> x (a != 0), also as two same-sign terms of a
    larger sum of additions and subtractions."""
    terms: List[Tuple[int, Expr]] = []
    _signed_terms(e, 1, terms)
    if len(terms) < 2:
        return None
    for i, (si, ti) in enumerate(terms):
        got = _scaled_floor(ti)
        if got is None:
            continue
        a, x = got
        for j, (sj, tj) in enumerate(terms):
            if j == i or sj != si or type(tj) is not Mod or tj.num != x or tj.den != a:
                continue
            if not prover.nonzero(a):
                return None
            rest = [(s, t) for k, (s, t) in enumerate(terms) if k not in (i, j)] + [(si, x)]
            acc = None
            for s, t in rest:
                if acc is None:
                    acc = t if s > 0 else Sub(IntConst(0), t)
                else:
                    acc = Add(acc, t) if s > 0 else Sub(acc, t)
            return acc
    return None


TABLE_RULES = (rule_mod_of_multiple_sum, rule_div_of_multiple_sum, rule_div_of_mod, rule_div_below_bound,
               rule_mod_below_bound, rule_div_by_one_assoc, rule_recompose)
