"""CUDA code generation for LEGO index expressions.

Turns a set of named output expressions over ranged input variables into one
``__device__ __forceinline__`` function:

* **CSE** -- expressions are DAGs (structural hashing in :mod:`.expr`); every
  distinct node becomes one typed temporary, so the anti-diagonal inverse's
  isqrt and selects are computed once instead of the tree's dozens of times.
* **Per-node integer width** from interval analysis (``simplify.Intervals``,
  the reference's ``range_of`` semantics): a node is ``int`` when its value
  range fits 32 bits, otherwise ``long long``.  Intervals cover the full
  variable ranges regardless of ``Select`` conditions, so computing both
  arms eagerly (straight-line, no divergence) can never overflow.
* **Floor semantics** (reference ``expr.py:285``/``:290``) without the C
  profile's silent non-negativity assumption (``emit.py:4-7``): non-negative
  numerators divide as unsigned (shift/mask for powers of two), possibly
  negative ones use arithmetic shift / mask (exact floor for 2^k) or the
  ``lego_fdiv``/``lego_fmod`` helpers.
* **Exact isqrt** via ``lego_isqrt`` (float sqrt plus integer fix-up).

The helpers live in ``csrc/lego_index.cuh``; generated code is spliced into
the kernel templates of ``csrc/remap_kernels.cuh`` and compiled for sm_100a.
"""

from __future__ import annotations

from typing import Dict, List, Mapping, Sequence, Tuple

from .errors import UnsupportedNode
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
    children,
    unique_nodes,
)
from .simplify import Intervals

I32_MIN, I32_MAX = -(1 << 31), (1 << 31) - 1
I64_MIN, I64_MAX = -(1 << 63), (1 << 63) - 1


def _fits32(r) -> bool:
    return I32_MIN <= r[0] and r[1] <= I32_MAX


def _pow2(d: int) -> int:
    return d.bit_length() - 1 if d > 0 and d & (d - 1) == 0 else -1


class DeviceFunction:
    """Generated source of one device function plus its signature facts."""

    def __init__(self, name: str, source: str, inputs: Sequence[str], outputs: Sequence[str],
                 out_types: Sequence[str], n_ops: int):
        self.name = name
        self.source = source
        self.inputs = list(inputs)
        self.outputs = list(outputs)
        self.out_types = list(out_types)
        self.n_ops = n_ops

    def __repr__(self):
        return f"DeviceFunction({self.name}, ops={self.n_ops})"


def generate(name: str, inputs: Sequence[Var], outputs: Mapping[str, Expr],
             bounds: Mapping[str, Tuple[int, int]] = None) -> DeviceFunction:
    """``static __device__ __forceinline__ void name(long long in..., T& out...)``.

    Inputs arrive as ``long long`` (the kernel's flat indices); each output
    is written through a reference of its own width.  ``bounds`` states true
    value ranges of outputs that interval analysis cannot prove (e.g. a
    layout inverse lands in [0, size) although its terms cancel); an output
    whose bound fits 32 bits lets the terms feeding it compute mod 2^32.
    """
    bounds = dict(bounds or {})
    iv = Intervals()
    for v in inputs:
        if v.range is None:
            raise UnsupportedNode(f"input {v.name} needs a range for code generation")
    order: List[Expr] = []
    seen = set()
    for e in outputs.values():
        for n in unique_nodes(e):
            if n not in seen:
                seen.add(n)
                order.append(n)
    # Modular narrowing: a node whose every use is an operand of +, -, * or a
    # Select arm, leading only to values that fit 32 bits, can be computed
    # mod 2^32 (ring homomorphism) in `unsigned` even when its own range does
    # not fit -- e.g. the anti-diagonal inverse's i*16383 terms that cancel.
    uses: Dict[Expr, List[Tuple[Expr, str]]] = {}

    def _cond_nodes(c, acc):
        if type(c) is Cmp:
            acc.extend([c.lhs, c.rhs])
        elif type(c) is And:
            _cond_nodes(c.lhs, acc)
            _cond_nodes(c.rhs, acc)

    for n in order:
        t = type(n)
        if t in (Add, Sub, Mul):
            for ch in (n.lhs, n.rhs):
                uses.setdefault(ch, []).append((n, "ring"))
        elif t is Select:
            for ch in (n.then, n.orelse):
                uses.setdefault(ch, []).append((n, "arm"))
            acc: List[Expr] = []
            _cond_nodes(n.cond, acc)
            for ch in acc:
                uses.setdefault(ch, []).append((n, "other"))
        else:
            for ch in children(n):
                uses.setdefault(ch, []).append((n, "other"))
    out_fits = {}
    for oname, e in outputs.items():
        fits = _fits32(iv.of(e)) or (oname in bounds and _fits32(bounds[oname]))
        out_fits[oname] = fits
        uses.setdefault(e, []).append((e, "out32" if fits else "other"))
    modsafe: Dict[Expr, bool] = {}

    def _modsafe(n) -> bool:
        if n in modsafe:
            return modsafe[n]
        modsafe[n] = False                      # cycle guard (DAGs have none)
        ok = bool(uses.get(n))
        for parent, role in uses.get(n, []):
            if role == "out32":
                continue
            if role not in ("ring", "arm") or not (_fits32(iv.of(parent)) or _modsafe(parent)):
                ok = False
                break
        modsafe[n] = ok
        return ok

    # conditions are not Exprs; generate their sub-expressions via Select
    names: Dict[Expr, str] = {}
    types: Dict[Expr, str] = {}
    lines: List[str] = []
    in_names = {v.name for v in inputs}
    for v in inputs:
        r = iv.of(v)
        t = "int" if _fits32(r) else "long long"
        names[v] = f"(({t}){v.name})"
        types[v] = t
    counter = [0]
    n_ops = 0

    def tmp(t: str, text: str, node: Expr) -> str:
        nm = f"t{counter[0]}"
        counter[0] += 1
        lines.append(f"  const {t} {nm} = {text};")
        names[node] = nm
        types[node] = t
        return nm

    def cast(node: Expr, t: str) -> str:
        s = names[node]
        return s if types[node] == t else f"(({t}){s})"

    def cond_text(c) -> str:
        if type(c) is Cmp:
            for side in (c.lhs, c.rhs):
                if side not in names:
                    emit(side)
            t = "long long" if "long long" in (types[c.lhs], types[c.rhs]) else "int"
            return f"({cast(c.lhs, t)} {c.op} {cast(c.rhs, t)})"
        if type(c) is And:
            return f"({cond_text(c.lhs)} && {cond_text(c.rhs)})"
        raise UnsupportedNode(f"cannot lower condition {type(c).__name__}")

    def emit(node: Expr):
        nonlocal n_ops
        if node in names:
            return
        for ch in children(node):
            emit(ch)
        t = type(node)
        r = iv.of(node)
        res_t = "int" if _fits32(r) else ("unsigned" if t in (Add, Sub, Mul, Select) and _modsafe(node)
                                          else "long long")
        if t is IntConst:
            v = node.value
            if _fits32((v, v)):
                names[node] = f"({v})"
                types[node] = "int"
            else:
                names[node] = f"({v}LL)"
                types[node] = "long long"
            return
        if t is Var:
            if node.name not in in_names:
                raise UnsupportedNode(f"free variable {node.name} is not an input")
            return
        n_ops += 1
        if t in (Add, Sub, Mul):
            op = {Add: "+", Sub: "-", Mul: "*"}[t]
            if res_t == "unsigned" or "int" != types[node.lhs] or "int" != types[node.rhs] and res_t == "int":
                if res_t == "long long":
                    tmp(res_t, f"{cast(node.lhs, res_t)} {op} {cast(node.rhs, res_t)}", node)
                else:   # wrapping 32-bit arithmetic (exact mod 2^32)
                    text = f"{cast(node.lhs, 'unsigned')} {op} {cast(node.rhs, 'unsigned')}"
                    tmp(res_t, text if res_t == "unsigned" else f"(int)({text})", node)
                return
            tmp(res_t, f"{cast(node.lhs, res_t)} {op} {cast(node.rhs, res_t)}", node)
            return
        if t is FloorDiv or t is Mod:
            is_div = t is FloorDiv
            num_r = iv.of(node.num)
            wide = "long long" if not _fits32(num_r) or res_t == "long long" else "int"
            if type(node.den) is IntConst and node.den.value > 0:
                d = node.den.value
                k = _pow2(d)
                if num_r[0] >= 0:
                    ut = "unsigned long long" if wide == "long long" else "unsigned"
                    num = f"(({ut}){cast(node.num, wide)})"
                    if k >= 0:
                        text = f"{num} >> {k}" if is_div else f"{num} & {d - 1}u"
                    else:
                        suf = "ull" if ut.startswith("unsigned long") else "u"
                        text = f"{num} {'/' if is_div else '%'} {d}{suf}"
                    tmp(res_t, f"({res_t})({text})", node)
                    return
                if k >= 0:
                    # arithmetic shift / two's-complement mask are exact floor ops
                    text = (f"{cast(node.num, wide)} >> {k}" if is_div
                            else f"{cast(node.num, wide)} & {d - 1}")
                    tmp(res_t, f"({res_t})({text})", node)
                    return
            helper = "lego_fdiv" if is_div else "lego_fmod"
            wd = "long long" if "long long" in (wide, types.get(node.den, "int")) else wide
            tmp(res_t, f"({res_t}){helper}({cast(node.num, wd)}, {cast(node.den, wd)})", node)
            return
        if t is Select:
            c = cond_text(node.cond)
            tmp(res_t, f"{c} ? {cast(node.then, res_t)} : {cast(node.orelse, res_t)}", node)
            return
        if t is Call:
            a = node.args[0]
            ar = iv.of(a)
            fn = "lego_isqrt32" if _fits32(ar) else "lego_isqrt64"
            at = "long long" if fn.endswith("64") else "int"
            tmp(res_t, f"({res_t}){fn}({cast(a, at)})", node)
            return
        raise UnsupportedNode(f"cannot lower {t.__name__}")

    for node in order:
        emit(node)
    out_types = []
    sig_in = ", ".join(f"const long long {v.name}" for v in inputs)
    sig_out = []
    body_out = []
    for oname, e in outputs.items():
        # outputs are always 64-bit in the signature; the value's own width
        # (int when it fits) is what the arithmetic above used
        out_types.append("long long")
        sig_out.append(f"long long& {oname}")
        if types.get(e) == "unsigned":          # wrapped value whose true range fits int
            body_out.append(f"  {oname} = (long long)(int){names[e]};")
        else:
            body_out.append(f"  {oname} = {cast(e, 'long long')};")
    sig = ", ".join([s for s in (sig_in, ", ".join(sig_out)) if s])
    src = (f"static __device__ __forceinline__ void {name}({sig}) {{\n"
           + "\n".join(lines + body_out) + "\n}\n")
    return DeviceFunction(name, src, [v.name for v in inputs], list(outputs), out_types, n_ops)


def constant(name: str, value: int) -> str:
    t = "int" if _fits32((value, value)) else "long long"
    suf = "" if t == "int" else "LL"
    return f"static constexpr {t} {name} = {value}{suf};\n"


def shape_tuple(values: Sequence[int]) -> Tuple[int, ...]:
    return tuple(int(v) for v in values)
