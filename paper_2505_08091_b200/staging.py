"""Box-staged gathers: proving that a gather reads one compact source box per
block of destination elements (multi-stage chains
whose last stage is an in-tile GenP, e.g. Eq. (2)'s tile-then-antidiag).

For ``dst[f] = src[g(f)]`` and a block size B the planner proves

    g(q*B + r) == base(q) + local(r)      for every q in [0, n/B), r in [0, B)

and then reads ``local`` as a box: R source rows of C consecutive elements at
row stride SX.  A CTA loads its block's box with coalesced 16-byte loads into
shared memory and writes the B destination elements as coalesced vectors,
reading the box through a per-layout offset table ``local(r) -> smem cell``
(LEGO_KIND 5 in ``csrc/remap_kernels.cuh``).

The proof is exact, not sampled:

1. substitute f = q*B + r and simplify;
2. every maximal sub-expression that depends on r alone is evaluated for all
   B values of r (a finite domain) and replaced by a fresh variable carrying
   its exact value range (a constant when the range is a single value) --
   this hands the simplifier the facts about isqrt/select-heavy in-tile
   arithmetic (e.g. the anti-diagonal inverse, reference layout.py:580-599)
   that interval analysis cannot derive;
3. simplify again and split the linear form into terms over q alone and
   terms over the r-atoms alone; any mixed term rejects the block size.

Everything is host-side, once per (layout pair, element size).
"""

from __future__ import annotations

import os
from typing import Dict, Optional, Tuple

import numpy as np

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
    eval_expr,
    variables,
)
from .simplify import Lin, _build, _lin_of, simplify

# block sizes tried (elements of the destination): the largest and smallest
BLOCKS = (16384, 8192, 4096, 2048, 1024, 512, 256)
# most block sizes tried per plan (each costs one simplification)
MAX_BLOCKS = 16
# shared-memory budget of one box (bytes)
BOX_SMEM = 48 * 1024
# preferred destination bytes per block (16 KiB: 8 resident CTAs per SM keep
# 128 KiB of loads in flight)
BOX_TARGET = int(os.environ.get("LEGO_BOX_TARGET", str(16 * 1024)))
# TMA-fed persistent staged kernel (cp.async.bulk box rows, double-buffered)
# when the box rows are provably 16-byte aligned.  Off by default: on the f1
# chain (256-byte box rows) it measured slower than the one-block-per-CTA
# kernel (int32 5579 vs 6196 GB/s, bf16 4378 vs 5407; scripts/quick_staged.py)
# -- 1-D bulk copies of a few hundred bytes do not amortise the TMA issue
BOX_BULK = int(os.environ.get("LEGO_BOX_BULK", "0"))
# threads per CTA of the staged kernel
BOX_THREADS = int(os.environ.get("LEGO_BOX_THREADS", "256"))
# smem-wavefront cost of one warp-wide global store in the store-mode model
STG_WEIGHT = 8
# store mode override for experiments: "" (cost model), "vec" or "scalar"
BOX_STORE = os.environ.get("LEGO_BOX_STORE", "")
# shortest box row worth staging (bytes): a 32-byte sector
MIN_ROW_BYTES = 32


# ---------------------------------------------------------------------------
# vectorised exact evaluation (int64 numpy; semantics of reference expr.py:261-316)
# ---------------------------------------------------------------------------

def _isqrt_vec(x: np.ndarray) -> np.ndarray:
    if np.any(x < 0):
        raise ValueError("isqrt of a negative value")
    r = np.floor(np.sqrt(x.astype(np.float64))).astype(np.int64)
    r = np.where(r * r > x, r - 1, r)
    r = np.where((r + 1) * (r + 1) <= x, r + 1, r)
    return r


def eval_vec(e: Expr, env: Dict[str, np.ndarray]) -> np.ndarray:
    """Evaluate e for every lane of the int64 arrays in env.  Select arms
    are both computed (a lane's unselected arm may be garbage but never
    reaches the result); division by zero in a selected arm raises."""
    memo: Dict[int, np.ndarray] = {}
    size = len(next(iter(env.values())))

    def ev(n):
        got = memo.get(id(n))
        if got is not None:
            return got
        t = type(n)
        if t is IntConst:
            v = np.full(size, n.value, dtype=np.int64)
        elif t is Var:
            v = np.asarray(env[n.name], dtype=np.int64)
        elif t is Add:
            v = ev(n.lhs) + ev(n.rhs)
        elif t is Sub:
            v = ev(n.lhs) - ev(n.rhs)
        elif t is Mul:
            v = ev(n.lhs) * ev(n.rhs)
        elif t in (FloorDiv, Mod):
            num, den = ev(n.num), ev(n.den)
            zero = den == 0
            safe = np.where(zero, 1, den)
            v = num // safe if t is FloorDiv else num % safe
            v = np.where(zero, 0, v)
            memo[id(n)] = v
            zeros[id(n)] = zero
            return v
        elif t is Select:
            c = cond(n.cond)
            v = np.where(c, ev(n.then), ev(n.orelse))
        elif t is Call:
            a = ev(n.args[0])
            v = _isqrt_vec(np.maximum(a, 0))
            negs[id(n)] = a < 0
        else:
            raise TypeError(f"not an expression: {n!r}")
        memo[id(n)] = v
        return v

    def cond(c):
        if type(c) is Cmp:
            a, b = ev(c.lhs), ev(c.rhs)
            return {"<": a < b, "<=": a <= b, "==": a == b, ">=": a >= b, ">": a > b}[c.op]
        return cond(c.lhs) & cond(c.rhs)

    zeros: Dict[int, np.ndarray] = {}
    negs: Dict[int, np.ndarray] = {}
    with np.errstate(all="ignore"):
        out = ev(e)
    if zeros or negs:
        # a lane that divided by zero (or took isqrt of a negative value)
        # must not depend on it: re-check such lanes with the exact scalar
        # evaluator, which raises where the reference would
        bad = np.zeros(size, dtype=bool)
        for m in list(zeros.values()) + list(negs.values()):
            bad |= m
        for k in np.nonzero(bad)[0][:64]:
            want = eval_expr(e, {name: int(a[k]) for name, a in env.items()})
            if want != int(out[k]):
                raise ValueError("vectorised evaluation disagrees with the exact evaluator")
        if bad.sum() > 64:
            raise ValueError("too many lanes divide by zero / take isqrt of a negative value")
    return out


# ---------------------------------------------------------------------------
# r-only atoms
# ---------------------------------------------------------------------------

def abstract_local(e: Expr, rname: str, rvals: np.ndarray) -> Tuple[Expr, Dict[str, Expr]]:
    """Replace every maximal sub-expression over ``rname`` alone (other than
    the bare variable) by an atom Var with its exact range over rvals (or by
    the constant it always equals).  Returns (new expr, atom name -> expr)."""
    vmemo: Dict[int, frozenset] = {}

    def fv(n) -> frozenset:
        got = vmemo.get(id(n))
        if got is None:
            t = type(n)
            if t is Var:
                got = frozenset((n.name,))
            elif t is IntConst:
                got = frozenset()
            else:
                got = frozenset().union(*(fv(x) for x in _kids(n)))
            vmemo[id(n)] = got
        return got

    atoms: Dict[Expr, Expr] = {}
    names: Dict[str, Expr] = {}
    memo: Dict[int, Expr] = {}

    def atom(n):
        got = atoms.get(n)
        if got is None:
            vals = eval_vec(n, {rname: rvals})
            lo, hi = int(vals.min()), int(vals.max())
            if lo == hi:
                got = IntConst(lo)
            else:
                name = f"_y{len(names)}"
                got = Var(name, VarRange(lo, hi + 1))
                names[name] = n
            atoms[n] = got
        return got

    def sub(n):
        got = memo.get(id(n))
        if got is not None:
            return got
        t = type(n)
        vs = fv(n)
        if t is IntConst or t is Var:
            out = n
        elif vs == frozenset((rname,)):
            out = atom(n)
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
        memo[id(n)] = out
        return out

    def cond(c):
        if type(c) is Cmp:
            return Cmp(c.op, sub(c.lhs), sub(c.rhs))
        return And(cond(c.lhs), cond(c.rhs))

    return sub(e), names


def _kids(n):
    t = type(n)
    if t in (Add, Sub, Mul, Cmp, And):
        return (n.lhs, n.rhs)
    if t in (FloorDiv, Mod):
        return (n.num, n.den)
    if t is Select:
        return (n.cond, n.then, n.orelse)
    if t is Call:
        return n.args
    raise TypeError(n)


# ---------------------------------------------------------------------------
# the plan
# ---------------------------------------------------------------------------

class BoxPlan:
    """g(q*B + r) == base(q) + row(r)*SX + col(r), box R x C (cell (0, 0) at
    base(q)), every cell read by the block (so every cell is a valid source
    element); ``offsets[r]`` = row(r)*pitch + col(r), the shared-memory cell."""

    def __init__(self, block, q, base, sx, rows, cols, pitch, offsets, vec_store, cost):
        self.block, self.q, self.base = block, q, base
        self.sx, self.rows, self.cols, self.pitch = sx, rows, cols, pitch
        self.offsets, self.vec_store, self.cost = offsets, vec_store, cost

    def __repr__(self):
        return (f"box {self.rows}x{self.cols} (stride {self.sx}, pitch {self.pitch}) per "
                f"{self.block} elements, {'vector' if self.vec_store else 'scalar'} stores")


def _separate(g: Expr, f: Var, n: int, block: int):
    """(q, base(q), local values over r) or None."""
    q = Var("q", VarRange(0, n // block))
    r = Var("r", VarRange(0, block))
    rvals = np.arange(block, dtype=np.int64)
    from .lower import substitute
    e = simplify(substitute(g, {f.name: q * block + r}))
    e, names = abstract_local(e, "r", rvals)
    e = simplify(e)
    lin = _lin_of(e)
    qpart, rpart = Lin({}, lin.const), Lin({}, 0)
    for a, c in lin.terms.items():
        vs = set(variables(a))
        if vs <= {"q"}:
            qpart.terms[a] = c
        elif "q" not in vs:
            rpart.terms[a] = c
        else:
            return None
    local = _build(rpart)
    env = {"r": rvals}
    for name, sube in names.items():
        env[name] = eval_vec(sube, {"r": rvals})
    vals = eval_vec(local, env) if rpart.terms else np.zeros(block, dtype=np.int64)
    return q, simplify(_build(qpart)), vals


def _wavefronts(words: np.ndarray) -> int:
    """Shared-memory wavefronts of warp instructions: words is (instr, 32) of
    4-byte word addresses; per instruction the max number of distinct words
    that fall into one bank."""
    total = 0
    for row in words:
        u = np.unique(row)
        total += int(np.bincount(u % 32, minlength=32).max())
    return total


def _smem_cost(offsets: np.ndarray, rows: int, cols: int, pitch: int, elem: int, vec_store: bool) -> int:
    v = 16 // elem
    # store phase: lane k of a warp reads element k*V + e (vector) or k (scalar)
    if vec_store:
        idx = offsets.reshape(-1, 32, v).transpose(0, 2, 1).reshape(-1, 32)
    else:
        idx = offsets.reshape(-1, 32)
    cost = _wavefronts(idx * elem // 4)
    # load phase: consecutive lanes own consecutive 16-byte vectors along box
    # rows (whole-vector rows) or consecutive cells (scalar loads); the
    # vectors go to shared memory whole when the pitch keeps 16-byte cells
    cells = np.arange(rows * cols, dtype=np.int64)
    addr = (cells // cols) * pitch + cells % cols
    if (cols * elem) % 16 == 0:
        if (pitch * elem) % 16 == 0:
            cost += -(-rows * cols * elem // 128)
        else:
            nvec = rows * cols // v
            a = addr[: (nvec // 32) * 32 * v].reshape(-1, 32, v).transpose(0, 2, 1).reshape(-1, 32)
            cost += _wavefronts(a * elem // 4)
    else:
        a = addr[: (len(addr) // 32) * 32].reshape(-1, 32)
        cost += _wavefronts(a * elem // 4)
    # global store instructions (one per 32 lanes), weighted as measured on
    # the f1 chain: 16-byte stores with 4-way conflicted smem reads beat
    # conflict-free scalar stores (int32 6191 vs 6082 GB/s, bf16 5391 vs
    # 4969, u8 3264 vs 2808; scripts/quick_staged.py)
    cost += STG_WEIGHT * (len(offsets) // 32) // (v if vec_store else 1)
    return cost


def box_plan(g: Expr, f: Var, n_dst: int, n_src: int, elem_bytes: int) -> Optional[BoxPlan]:
    if elem_bytes not in (1, 2, 4, 8) or n_dst < 256:
        return None
    v = 16 // elem_bytes
    # blocks whose destination bytes fit BOX_TARGET first (largest first),
    # then larger ones (smallest first) up to the shared-memory budget
    # candidates: every multiple of 32 in [256, 16384] dividing n_dst (tiles of
    # 24 x 16 or 48 x 48 elements give blocks like 384 or 2304), at most
    # MAX_BLOCKS of them
    cands = [b for b in range(BLOCKS[-1], BLOCKS[0] + 1, 32) if n_dst % b == 0]
    fits = sorted((b for b in cands if b * elem_bytes <= BOX_TARGET), reverse=True)
    order = (fits + sorted(b for b in cands if b * elem_bytes > BOX_TARGET))[:MAX_BLOCKS]
    for block in order:
        if n_dst % block or block > n_dst:
            continue
        try:
            sep = _separate(g, f, n_dst, block)
        except Exception:              # noqa: BLE001 -- any failure just rejects this block size
            sep = None
        if sep is None:
            continue
        q, base, vals = sep
        lo = int(vals.min())
        w = vals - lo
        if np.array_equal(w, np.arange(block)):
            return None                        # in-order contiguous: the vector gather is exact
        u = np.unique(w)
        breaks = np.nonzero(np.diff(u) != 1)[0]
        starts = u[np.r_[0, breaks + 1]]       # starts[0] == 0
        sx = int(u[-1]) + 1 if len(starts) == 1 else int(np.gcd.reduce(starts[1:]))
        rowv, col = w // sx, w % sx
        c0 = int(col.min())
        col = col - c0
        cols, rows = int(col.max()) + 1, int(rowv.max()) + 1
        if rows * cols * elem_bytes > BOX_SMEM or cols * elem_bytes < MIN_ROW_BYTES:
            continue
        if len(u) != rows * cols:
            continue                           # every box cell must be a source element the block reads
        best = None
        for pad in range(0, 9):
            pitch = cols + pad
            if rows * pitch * elem_bytes > BOX_SMEM:
                break
            offs = rowv * pitch + col
            for vec_store in (True, False):
                if vec_store and block % (32 * v):
                    continue
                if BOX_STORE and vec_store != (BOX_STORE == "vec"):
                    continue
                cost = _smem_cost(offs, rows, cols, pitch, elem_bytes, vec_store)
                if best is None or cost < best[0]:
                    best = (cost, pitch, offs, vec_store)
        if best is None:
            continue
        cost, pitch, offs, vec_store = best
        base = simplify(Add(base, IntConst(lo + c0)))
        return BoxPlan(block, q, base, sx, rows, cols, pitch, offs, vec_store, cost)
    return None
