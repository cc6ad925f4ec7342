"""Bulk layout operations on B200 -- the backend's data-parallel hot path.

The reference evaluates a layout one index at a time in Python
(``GroupBy.apply``/``inv``, ``pkg/src/lego/layout.py:313-328``; ~10-15 us per
element).  Here a layout is lowered once (:mod:`.lower`), its index
arithmetic generated as CUDA (:mod:`.codegen`), spliced into a hand-written
kernel template (``csrc/remap_kernels.cuh``), JIT-compiled for sm_100a by
NVRTC (cubins cached on disk) and launched through the C ABI.

Public operations (torch tensors in, torch tensors out, all on the GPU):

* :func:`apply_map` / :func:`inv_map` -- a layout's bijection over its whole
  index space (the reference's per-element ``apply`` / ``inv`` in bulk);
* :func:`remap` (and :func:`gather` / :func:`scatter`) -- move a tensor from
  one layout to another: for every logical index x,
  ``dst[dst.apply(x)] = src[src.apply(x)]``;
* :func:`check_bijective` -- prove a layout is a permutation on the device
  (``validate`` only enumerates GenPs up to 4096 points);
* :func:`softmax`, :func:`nw_score`, :func:`gemm` -- the fixed kernels.

No function here computes on the CPU; without the native library they raise
:class:`~.errors.BackendUnavailable`.
"""

from __future__ import annotations

import ctypes
import os
import threading
from typing import Dict, Optional, Tuple

from . import codegen, lower, runtime, staging
from .errors import BijectivityViolation, LegoError, ShapeMismatch, UnsupportedNode
from .expr import IntConst, Var, VarRange
from .simplify import _lin_of

CSRC = os.path.join(os.path.dirname(os.path.abspath(__file__)), "csrc")
_TEXT: Dict[str, str] = {}

# kernel launches issued through this module since import (for bench.py's
# gpu_launches count; the driver cross-checks with the loaded .so list)
LAUNCHES = [0]


def _text(name: str) -> str:
    if name not in _TEXT:
        with open(os.path.join(CSRC, name)) as fh:
            _TEXT[name] = fh.read()
    return _TEXT[name]


def _assemble(gen_body: str, defines: Dict[str, int]) -> str:
    """Program source: helpers + generated namespace + kernel templates."""
    defines = {**defines, **({"LEGO_LDV": LOAD_HINT} if LOAD_HINT else {}),
               **({"LEGO_STV": STORE_HINT} if STORE_HINT else {})}
    head = "".join(f"#define {k} {v}\n" for k, v in defines.items())
    return (head + _text("lego_index.cuh").replace("#pragma once", "") + "\nnamespace gen {\n"
            + gen_body + "}\n" + _text("remap_kernels.cuh").replace("#pragma once", ""))


def _layout_key(layout) -> tuple:
    return (type(layout).__name__, layout) if layout is not None else ("row",)


# ---------------------------------------------------------------------------
# program builders
# ---------------------------------------------------------------------------

class _ProgramCache:
    """Loaded programs, per device.  Two levels: (layout key, device) ->
    program (an LRU: layouts holding user GenPs compare by closure identity,
    so every fresh parse is a new key) and (source SHA-256, device) ->
    program, so re-planning an equal layout reuses the loaded module instead
    of loading another.  A program is published only once complete."""

    def __init__(self, limit: int = 256):
        from collections import OrderedDict
        self.limit = limit
        self.by_key = OrderedDict()
        self.by_source: Dict[tuple, runtime.Program] = {}
        self.lock = threading.Lock()

    def get(self, key, builder, device: int):
        k = key + (device,)
        with self.lock:
            prog = self.by_key.get(k)
            if prog is not None:
                self.by_key.move_to_end(k)
                return prog
        source, info, extra = builder()
        import hashlib
        # a loaded program is shared only between builds with the same text,
        # geometry and plan facts (e.g. NW programs of equal text for two n)
        facts = tuple(getattr(info, f) for f, _t in info._fields_)
        plain = tuple(sorted((k, v) for k, v in (extra or {}).items() if isinstance(v, (int, str, bool))))
        sk = (hashlib.sha256(source.encode()).hexdigest(), facts, plain, device)
        with self.lock:
            prog = self.by_source.get(sk)
        if prog is None:
            import torch
            cubin = runtime.compile_cubin(source)
            with torch.cuda.device(device):
                prog = runtime.Program(cubin, info, source)
            for name, value in (extra or {}).items():
                setattr(prog, name, value)
        with self.lock:
            prog = self.by_source.setdefault(sk, prog)
            self.by_key[k] = prog
            self.by_key.move_to_end(k)
            while len(self.by_key) > self.limit:
                _old_key, old = self.by_key.popitem(last=False)
                if not any(p is old for p in self.by_key.values()):
                    self.by_source = {kk: pp for kk, pp in self.by_source.items() if pp is not old}
        return prog


_CACHE = _ProgramCache()


def _program(key, builder, device: int):
    """builder() -> (source, info) or (source, info, {attr: value})."""
    def build():
        got = builder()
        return got if len(got) == 3 else (got[0], got[1], None)
    return _CACHE.get(key, build, device)


def index_map_source(layout) -> Tuple[str, runtime.ProgramInfo]:
    check_genp_agreement(layout)
    x, app = lower.apply_map_expr(layout)
    injective = getattr(lower._group(layout), "injective", False)
    defines = {"LEGO_KIND": 0}
    body = codegen.constant("N", lower.logical_size(layout))
    body += codegen.constant("M", lower.physical_size(layout))
    body += codegen.generate("apply_fn", [x], {"out": app},
                             bounds={"out": (-1, lower.physical_size(layout) - 1)}).source
    if injective:
        body += "static __device__ __forceinline__ void inv_fn(const long long f, long long& out) { out = -1; }\n"
    else:
        f, inv = lower.inv_map_expr(layout)
        body += codegen.generate("inv_fn", [f], {"out": inv},
                                 bounds={"out": (0, lower.logical_size(layout) - 1)}).source
        side = lower.antidiag_side(layout)
        if INV_RUNS and side is not None and side > 1 and lower.diagonal_runs_contiguous(layout, side):
            body += codegen.constant("RUN_N", side)
            defines["LEGO_INV_RUNS"] = INV_RUNS
    # positions of an injective-mode layout may run past its logical size
    units = lower.value_range(app)[1] + 1 if injective else lower.physical_size(layout)
    info = runtime.ProgramInfo(kind=runtime.KIND_INDEX_MAP, elem_bytes=0,
                               n=lower.logical_size(layout), units=max(units, 1),
                               unit_threads=1, block=256, smem_bytes=0)
    return _assemble(body, defines), info


# source vectors per thread of the fused fill scatter
FILL_UNROLL = int(os.environ.get("LEGO_FILL_UNROLL", "1"))   # measured: 1 121.0 us, 2 121.4, 4 123.1
# the run-walking inverse map of anti-diagonal layouts (0 disables it)
INV_RUNS = int(os.environ.get("LEGO_INV_RUNS", "1"))


class RemapPlan:
    """What the lowering decided for one (src layout, dst layout, elem size)."""

    def __init__(self, kind, n_dst, n_src, elem_bytes, contig, masked, source, info, detail):
        self.kind, self.n_dst, self.n_src = kind, n_dst, n_src
        self.elem_bytes, self.contig, self.masked = elem_bytes, contig, masked
        self.source, self.info, self.detail = source, info, detail

    def __repr__(self):
        names = {1: "gather", 2: "transpose", 3: "band", 4: "scatter", 5: "staged"}
        if "interleave" in self.detail:
            names = {**names, 2: "interleave"}
        return (f"RemapPlan({names[self.kind]}, n={self.n_dst}, elem={self.elem_bytes}B, "
                f"{self.detail})")


class Route:
    """Destination routing of a remap over several buffers: destination
    element v goes to buffer ``peer(v)`` at element offset ``off(v)``.
    ``fn(v: Var) -> (peer_expr, off_expr)`` builds both as LEGO index
    expressions; ``key`` identifies the routing for the program cache."""

    def __init__(self, world: int, fn, key):
        self.world, self.fn, self.key = world, fn, key


def plan_remap(src_layout, dst_layout, elem_bytes: int, route: Optional[Route] = None,
               fill: bool = False) -> RemapPlan:
    """``fill``: scatters into injective layouts write every destination
    position (unhit ones with a fill value); other kinds write every
    position anyway and ignore it."""
    if elem_bytes not in (1, 2, 4, 8, 16):
        raise UnsupportedNode(f"element size {elem_bytes} not supported (1, 2, 4, 8 or 16 bytes)")
    check_genp_agreement(src_layout)
    check_genp_agreement(dst_layout)
    if route is not None:
        return _routed_plan(src_layout, dst_layout, elem_bytes, route)
    band = _band_plan(src_layout, dst_layout, elem_bytes)
    if band is not None:
        return band
    scatter = _scatter_plan(src_layout, dst_layout, elem_bytes, fill)
    if scatter is not None:
        return scatter
    f, g, n_dst, n_src = lower.gather_expr(src_layout, dst_layout)
    lo, _hi = lower.value_range(g)
    masked = lo < 0
    vec = 16 // elem_bytes
    if n_dst % vec:
        return _scalar_gather_plan(f, g, n_dst, n_src, elem_bytes, masked)
    if not masked:
        variant = TRANSPOSE_VARIANT or ("smem" if elem_bytes == 1 else "regT")
        smem_variant = variant == "smem"
        persist = variant == "persist"
        xmajor = variant == "regT"
        tpw = 2 if variant == "reg2" else 1
        xv, yv = (8, 8) if smem_variant else ((8, 4) if xmajor else (4, 8))
        tp = lower.transpose_plan(g, f, n_dst, elem_bytes, xv, yv, TILE_ORDER)
        if tp is not None:
            body = codegen.constant("N", n_dst) + codegen.constant("TILES", tp.tiles)
            body += codegen.constant("SX", tp.sx) + codegen.constant("DY", tp.dy)
            body += codegen.generate("origin", [tp.t], {"f0": tp.origin_f0,
                                                        "s0": tp.origin_s0}).source
            warps = 4 if smem_variant else (TRANSPOSE_WARPS or _TRANSPOSE_WARPS_BY_ELEM[elem_bytes])
            v = 16 // elem_bytes
            smem = warps * 8 * v * 8 * 16 if smem_variant else 0
            per_cta = warps * tpw
            units = (tp.tiles + per_cta - 1) // per_cta
            if persist:
                units = min(units, PERSIST_CTAS)
            info = runtime.ProgramInfo(kind=runtime.KIND_TRANSPOSE, elem_bytes=elem_bytes, n=n_dst,
                                       units=units, unit_threads=32, block=32 * warps,
                                       smem_bytes=smem)
            src = _assemble(body, {"LEGO_KIND": 2, "LEGO_ELEM": elem_bytes,
                                   "LEGO_SMEM": int(smem_variant), "LEGO_TPW": tpw,
                                   "LEGO_PERSIST": int(persist), "LEGO_XMAJOR": int(xmajor),
                                   "LEGO_MINB": TRANSPOSE_MINB, "LEGO_TBLOCK": 32 * warps})
            return RemapPlan(runtime.KIND_TRANSPOSE, n_dst, n_src, elem_bytes, False, False, src,
                             info, f"tile {tp.tx}x{tp.ty} {variant}, SX={tp.sx}, DY={tp.dy}")
    if not masked and NARROW:
        npl = lower.narrow_plan(g, f, n_dst, elem_bytes)
        if npl is not None:
            return _narrow_remap_plan(npl, n_dst, n_src, elem_bytes)
    width = 1 if masked else lower.contiguous_width(g, f, n_dst, widths=(vec,))
    contig = width >= vec
    if not contig and BOX_STAGING:
        bp = staging.box_plan(g, f, n_dst, n_src, elem_bytes) if not masked else None
        if bp is not None:
            return _staged_plan(bp, n_dst, n_src, elem_bytes)
        if _mirrorable(src_layout, dst_layout):
            # the mirrored form: h = g^-1 maps source positions to destination
            # positions; source blocks land in destination boxes
            fh, h, _, _ = lower.gather_expr(dst_layout, src_layout)
            bp = staging.box_plan(h, fh, n_src, n_dst, elem_bytes)
            if bp is not None:
                return _staged_plan(bp, n_dst, n_src, elem_bytes, scatter=True)
    if contig and (n_src * elem_bytes) % 16:
        # 16-byte source vectors would straddle batch entries
        return _scalar_gather_plan(f, g, n_dst, n_src, elem_bytes, masked)
    body = codegen.constant("N", n_dst)
    body += codegen.generate("src_of", [f], {"s": g}, bounds={"s": (-1, n_src - 1)}).source
    unroll = 4
    block = 256
    nvec = n_dst // vec
    units = (nvec + block * unroll - 1) // (block * unroll)
    info = runtime.ProgramInfo(kind=runtime.KIND_GATHER, elem_bytes=elem_bytes, n=n_dst,
                               units=units, unit_threads=1, block=block, smem_bytes=0,
                               reserved=0 if contig else runtime.ALIGN_SRC_FREE)
    src = _assemble(body, {"LEGO_KIND": 1, "LEGO_ELEM": elem_bytes, "LEGO_CONTIG": int(contig),
                           "LEGO_MASKED": int(masked), "LEGO_UNROLL": unroll})
    return RemapPlan(runtime.KIND_GATHER, n_dst, n_src, elem_bytes, contig, masked, src, info,
                     f"contiguous={contig}, masked={masked}")


def _narrow_remap_plan(npl, n_dst, n_src, elem_bytes) -> RemapPlan:
    """Register interleave for a small innermost span (LEGO_KIND 2,
    LEGO_NARROW 1/2; lower.narrow_plan)."""
    vec = 16 // elem_bytes
    rng = (0, n_dst - 1)
    body = codegen.constant("N", n_dst) + codegen.generate("map", [npl.var], {"pos": npl.map},
                                                           bounds={"pos": rng}).source
    units = (n_dst // vec + 255) // 256
    info = runtime.ProgramInfo(kind=runtime.KIND_TRANSPOSE, elem_bytes=elem_bytes, n=n_dst, units=units,
                               unit_threads=1, block=256, smem_bytes=0, reserved=0)
    src = _assemble(body, {"LEGO_KIND": 2, "LEGO_ELEM": elem_bytes, "LEGO_NARROW": npl.mode, "LEGO_NY": npl.small})
    side = "source" if npl.mode == 1 else "destination"
    return RemapPlan(runtime.KIND_TRANSPOSE, n_dst, n_src, elem_bytes, False, False, src, info,
                     f"interleave: {side}-innermost span {npl.small}, {16 // npl.small}-byte chunks in registers")


def _routed_plan(src_layout, dst_layout, elem_bytes, route) -> RemapPlan:
    """A gather or register transpose whose 16-byte destination vectors are
    routed to peer buffers (remap_kernels.cuh LEGO_ROUTED).  Proves, for every
    aligned vector v = V*q + k (k < V), that peer(v) == peer(V*q),
    off(v) == off(V*q) + k and off(V*q) % V == 0, and 0 <= peer < world."""
    f, g, n_dst, n_src = lower.gather_expr(src_layout, dst_layout)
    vec = 16 // elem_bytes
    peer_e, off_e = (lower.simplify(lower.as_expr(e)) for e in route.fn(f))
    lo, hi = lower.value_range(g)
    if n_dst % vec or lo < 0:
        raise UnsupportedNode("routed remaps need whole 16-byte destination vectors and no masked reads")
    q = Var("q", VarRange(0, n_dst // vec))
    r = Var("r", VarRange(0, vec))
    at = lambda e, x: lower.simplify(lower.substitute(e, {f.name: x}))  # noqa: E731
    p0, o0 = at(peer_e, q * vec), at(off_e, q * vec)
    same_peer = lower.simplify(at(peer_e, q * vec + r) - p0) == IntConst(0)
    contiguous = lower.simplify(at(off_e, q * vec + r) - o0 - r) == IntConst(0)
    lin = _lin_of(o0)
    aligned = lin.const % vec == 0 and all(c % vec == 0 for c in lin.terms.values())
    plo, phi = lower.value_range(peer_e)
    if not (same_peer and contiguous and aligned and plo >= 0 and phi < route.world):
        raise UnsupportedNode("routing must keep each 16-byte destination vector in one peer, "
                              "contiguous and aligned")
    body = codegen.constant("N", n_dst)
    body += codegen.generate("route", [f], {"peer": peer_e, "off": off_e}).source
    tp = lower.transpose_plan(g, f, n_dst, elem_bytes, 8, 4, TILE_ORDER)
    if tp is not None:
        body += codegen.constant("TILES", tp.tiles) + codegen.constant("SX", tp.sx)
        body += codegen.constant("DY", tp.dy)
        body += codegen.generate("origin", [tp.t], {"f0": tp.origin_f0, "s0": tp.origin_s0}).source
        info = runtime.ProgramInfo(kind=runtime.KIND_TRANSPOSE, elem_bytes=elem_bytes, n=n_dst,
                                   units=(tp.tiles + 7) // 8, unit_threads=32, block=256, smem_bytes=0)
        src = _assemble(body, {"LEGO_KIND": 2, "LEGO_ELEM": elem_bytes, "LEGO_XMAJOR": 1,
                               "LEGO_MINB": TRANSPOSE_MINB, "LEGO_ROUTED": 1})
        return RemapPlan(runtime.KIND_TRANSPOSE, n_dst, n_src, elem_bytes, False, False, src, info,
                         f"routed over {route.world} peers, tile {tp.tx}x{tp.ty} regT")
    width = lower.contiguous_width(g, f, n_dst, widths=(vec,))
    contig = width >= vec
    body += codegen.generate("src_of", [f], {"s": g}, bounds={"s": (0, n_src - 1)}).source
    units = (n_dst // vec + 1023) // 1024
    info = runtime.ProgramInfo(kind=runtime.KIND_GATHER, elem_bytes=elem_bytes, n=n_dst,
                               units=units, unit_threads=1, block=256, smem_bytes=0,
                               reserved=0 if contig else runtime.ALIGN_SRC_FREE)
    src = _assemble(body, {"LEGO_KIND": 1, "LEGO_ELEM": elem_bytes, "LEGO_CONTIG": int(contig),
                           "LEGO_MASKED": 0, "LEGO_UNROLL": 4, "LEGO_ROUTED": 1})
    return RemapPlan(runtime.KIND_GATHER, n_dst, n_src, elem_bytes, contig, False, src, info,
                     f"routed over {route.world} peers, contiguous={contig}")


def _mirrorable(src_layout, dst_layout) -> bool:
    """Both sides are bijections with an inverse (no ExpandBy holes, no
    injective-only layout), so the source -> destination map exists."""
    for side in (src_layout, dst_layout):
        if isinstance(side, lower.ExpandBy):
            return False
        if side is not None and getattr(lower._group(side), "injective", False):
            return False
    return src_layout is not None


def _staged_plan(bp, n_dst, n_src, elem_bytes, scatter=False) -> RemapPlan:
    """Box-staged remap (LEGO_KIND 5): one CTA per destination block of
    bp.block elements with its source box staged through shared memory, or
    (scatter) one CTA per source block landing in its destination box."""
    v = 16 // elem_bytes
    cells = bp.rows * bp.pitch
    tab_t = "unsigned short" if cells <= 0xFFFF else "unsigned int"
    body = codegen.constant("B", bp.block) + codegen.constant("R", bp.rows)
    body += codegen.constant("C", bp.cols) + codegen.constant("PITCH", bp.pitch)
    body += codegen.constant("SX", bp.sx)
    body += f"typedef {tab_t} tab_t;\n"
    body += (f"__device__ __align__(32) const tab_t TAB[{bp.block}] = {{"
             + ",".join(str(int(o)) for o in bp.offsets) + "};\n")
    body += codegen.generate("base_of", [bp.q], {"b": bp.base}).source
    lvec = (bp.cols * elem_bytes) % 16 == 0 and (bp.sx * elem_bytes) % 16 == 0
    smem = -(-cells * elem_bytes // 16) * 16
    free = runtime.ALIGN_SRC_FREE | runtime.ALIGN_DST_FREE
    # TMA-fed persistent form: every box row a 16-byte-aligned bulk copy
    lin = _lin_of(bp.base)
    bulk = (staging.BOX_BULK and not scatter and lvec and (bp.pitch * elem_bytes) % 16 == 0
            and (lin.const * elem_bytes) % 16 == 0
            and all((c * elem_bytes) % 16 == 0 for c in lin.terms.values()))
    if bulk:
        boxb = -(-cells * elem_bytes // 128) * 128
        smem = 2 * boxb + 16
        per_sm = max(1, min(8, (220 * 1024) // (smem + 1024)))
        units = min(n_dst // bp.block, 148 * per_sm)
        reserved = runtime.ALIGN_SRC_FREE | (0 if bp.vec_store else runtime.ALIGN_DST_FREE)
        body += codegen.constant("N", n_dst)
    elif scatter:
        units, reserved = n_src // bp.block, free
    else:
        units = n_dst // bp.block
        reserved = runtime.ALIGN_SRC_FREE | (0 if bp.vec_store else runtime.ALIGN_DST_FREE)
    info = runtime.ProgramInfo(kind=runtime.KIND_STAGED, elem_bytes=elem_bytes, n=n_dst,
                               units=units, unit_threads=staging.BOX_THREADS, block=staging.BOX_THREADS,
                               smem_bytes=smem,
                               reserved=reserved)
    src = _assemble(body, {"LEGO_KIND": 5, "LEGO_ELEM": elem_bytes, "LEGO_LVEC": int(lvec),
                           "LEGO_SVEC16": int((bp.pitch * elem_bytes) % 16 == 0),
                           "LEGO_VSTORE": int(bp.vec_store), "LEGO_SCATTER": int(scatter),
                           "LEGO_BULK": int(bulk), "LEGO_BT": staging.BOX_THREADS})
    return RemapPlan(runtime.KIND_STAGED, n_dst, n_src, elem_bytes, False, False, src, info,
                     ("source blocks into destination " if scatter else "") + repr(bp)
                     + (", TMA bulk rows, persistent" if bulk else ""))


def _scalar_gather_plan(f, g, n_dst, n_src, elem_bytes, masked) -> RemapPlan:
    """Ragged sizes (n_dst not a whole number of 16-byte vectors, or source
    batch strides that are not 16-byte multiples): one element per thread."""
    body = codegen.constant("N", n_dst) + codegen.generate("src_of", [f], {"s": g},
                                                            bounds={"s": (-1, n_src - 1)}).source
    units = max(1, min((n_dst + 255) // 256, 148 * 16))
    info = runtime.ProgramInfo(kind=runtime.KIND_GATHER, elem_bytes=elem_bytes, n=n_dst,
                               units=units, unit_threads=1, block=256, smem_bytes=0,
                               reserved=runtime.ALIGN_SRC_FREE | runtime.ALIGN_DST_FREE)
    src = _assemble(body, {"LEGO_KIND": 1, "LEGO_ELEM": elem_bytes, "LEGO_SCALAR": 1,
                           "LEGO_MASKED": int(masked)})
    return RemapPlan(runtime.KIND_GATHER, n_dst, n_src, elem_bytes, False, masked, src, info,
                     f"scalar (ragged), masked={masked}")


# band tile (rows x anti-diagonals); static smem BR x (BK+1) elements must stay <= 48 KiB.
# 0 = measured default per direction (scripts/quick_band.py, 16384^2 int32 on B200):
# scatter (row-major -> antidiag) 128 x 32, gather 128 x 64
BAND_ROWS = int(os.environ.get("LEGO_BAND_ROWS", "0"))
BAND_DIAGS = int(os.environ.get("LEGO_BAND_DIAGS", "0"))
# transpose kernel variant: "reg" (register micro-tiles, 128-byte src runs,
# 64-byte dst runs), "regT" (the same with 128-byte dst runs, 64-byte src
# runs), "reg2" (two tiles per warp in flight), "persist" (persistent,
# cross-tile prefetch) or "smem" (128-byte runs on both sides through
# swizzled shared memory); empty = measured best on B200
# (scripts/quick_transpose.py, profiles/r01_transpose_variants.md): regT,
# with smem for 1-byte elements
TRANSPOSE_VARIANT = os.environ.get("LEGO_TRANSPOSE", "")
# load / store cache-hint variants of the remap kernels (remap_kernels.cuh LEGO_LDV / LEGO_STV)
# (measured: L2::256B sector promotion on loads, LEGO_LDV=1, +2.7% on the
# headline transpose and +1.4% on the tiled gather; scripts/quick_hints.py)
LOAD_HINT = int(os.environ.get("LEGO_LDV", "1"))
STORE_HINT = int(os.environ.get("LEGO_STV", "0"))
# warps per CTA of the register transpose; 0 = measured default per element
# size (scripts/quick_transpose_warps2.py, 16384^2 on B200: bf16 12 warps
# 170.0 us vs 8 warps 172.7; fp32 16 warps; int64 8)
TRANSPOSE_WARPS = int(os.environ.get("LEGO_TRANSPOSE_WARPS", "0"))
_TRANSPOSE_WARPS_BY_ELEM = {1: 8, 2: 12, 4: 16, 8: 8, 16: 8}
# minimum resident CTAs per SM requested for the register transpose (register cap)
TRANSPOSE_MINB = int(os.environ.get("LEGO_TRANSPOSE_MINB", "1"))
# warp-tile walk order of the transpose ("x", "y" or "block", see lower.transpose_plan)
TILE_ORDER = os.environ.get("LEGO_TILE_ORDER", "block")
# CTAs of the persistent transpose variant (2 resident CTAs x 148 SMs by default)
PERSIST_CTAS = int(os.environ.get("LEGO_PERSIST_CTAS", str(2 * 148)))
# register interleaves for digit permutations with a small innermost span (0 disables)
NARROW = int(os.environ.get("LEGO_NARROW", "1"))
# box-staged gathers (staging.py, LEGO_KIND 5) for non-contiguous gathers whose
# destination blocks each read one compact source box (0 disables)
BOX_STAGING = int(os.environ.get("LEGO_BOX", "1"))
# warps per band CTA (BR and BK must be multiples of it)
BAND_WARPS = int(os.environ.get("LEGO_BAND_WARPS", "8"))
# band tile order: 0 row-block major, 1 diagonal-block major, -1 = per direction
BAND_ORDER = int(os.environ.get("LEGO_BAND_ORDER", "-1"))


def _band_plan(src_layout, dst_layout, elem_bytes) -> Optional[RemapPlan]:
    """Row-major <-> anti-diagonal layout: band tiles (LEGO_KIND 3)."""
    if elem_bytes not in (1, 2, 4, 8):
        return None
    if src_layout is None and dst_layout is not None:
        side, direction = dst_layout, 0
    elif dst_layout is None and src_layout is not None:
        side, direction = src_layout, 1
    else:
        return None
    n = lower.antidiag_side(side)
    br = BAND_ROWS or 128
    bk = BAND_DIAGS or (32 if direction == 0 else 64)
    if br * (bk + 1) * elem_bytes > 48 * 1024:
        br, bk = 64, 64
    if n is not None and n % br:
        br, bk = 64, 64
    if n is None or n % br or n * n >= 2 ** 31 or not lower.diagonal_runs_contiguous(side, n):
        return None
    x = lower.flat_var("x", n * n)
    pos = lower.simplify(lower.as_expr(lower.apply_flat(side, x)))
    kblocks = (n + br + bk - 2) // bk + 1
    body = codegen.constant("NN", n) + codegen.constant("KBLOCKS", kblocks)
    body += codegen.generate("pos_of", [x], {"p": pos}, bounds={"p": (0, n * n - 1)}).source
    order = BAND_ORDER if BAND_ORDER >= 0 else (1 if direction == 0 else 0)
    if order == 0:
        units = (n // br) * kblocks
    else:
        units = ((2 * n - 1 + bk - 1) // bk) * (n // br)
    bw = BAND_WARPS
    info = runtime.ProgramInfo(kind=runtime.KIND_BAND, elem_bytes=elem_bytes, n=n * n, units=units,
                               unit_threads=32 * bw, block=32 * bw, smem_bytes=0,
                               reserved=runtime.ALIGN_SRC_FREE | runtime.ALIGN_DST_FREE)
    src = _assemble(body, {"LEGO_KIND": 3, "LEGO_ELEM": elem_bytes, "LEGO_DIR": direction,
                           "LEGO_BAND_ORDER": order, "LEGO_BR": br, "LEGO_BK": bk, "LEGO_BW": bw})
    return RemapPlan(runtime.KIND_BAND, n * n, n * n, elem_bytes, False, False, src, info,
                     f"band {br} rows x {bk} diagonals, order {order}, "
                     f"{'scatter' if direction == 0 else 'gather'}")


def _affine(e, x: Var, n: int):
    """(k, c) with e(x) == k*x + c for every x in [0, n), else None."""
    if n < 2:
        return None
    c = lower.value_at(e, x, 0)
    k = lower.value_at(e, x, 1) - c
    if c is None or k < 1:
        return None
    return (k, c) if lower.simplify(e - (x * k + c)) == IntConst(0) else None


def _scatter_plan(src_layout, dst_layout, elem_bytes, fill=False) -> Optional[RemapPlan]:
    """Row-major source into an injective-mode layout (no inverse exists):
    a true scatter, dst[apply(x)] = src[x] (LEGO_KIND 4).  With ``fill``
    every destination position is written: affine maps apply(x) = k*x + c
    (proven symbolically) get one kernel assembling whole 16-byte windows in
    registers; others a vector fill pass ahead of the scatter."""
    if src_layout is not None or dst_layout is None:
        return None
    if not getattr(lower._group(dst_layout), "injective", False):
        return None
    if elem_bytes not in (1, 2, 4, 8):
        raise UnsupportedNode("scatter supports 1, 2, 4 or 8-byte elements")
    x, app = lower.apply_map_expr(dst_layout)
    n_src = lower.logical_size(dst_layout)
    vec = 16 // elem_bytes
    scalar = n_src % vec != 0                               # ragged: one element per thread
    n_dst = lower.value_range(app)[1] + 1                   # highest position + 1
    body = codegen.constant("N", n_src) + codegen.constant("N_DST", n_dst)
    body += codegen.generate("pos_of", [x], {"p": app}).source
    units = max(1, min((n_src + 255) // 256, 148 * 16)) if scalar else (n_src // vec + 255) // 256
    reserved = runtime.ALIGN_DST_FREE | (runtime.ALIGN_SRC_FREE if scalar else 0)
    defines = {"LEGO_KIND": 4, "LEGO_ELEM": elem_bytes, "LEGO_SCALAR": int(scalar), "LEGO_FILL": int(fill)}
    detail = f"scatter into an injective layout, {n_dst} positions"
    if fill:
        aff = None if scalar else _affine(app, x, n_src)
        if aff is not None and (aff[1] * elem_bytes) % 16 == 0:
            k, c = aff
            defines.update({"LEGO_FK": k, "LEGO_FC": c})
            units = max((n_src // vec + 256 * FILL_UNROLL - 1) // (256 * FILL_UNROLL), (-(-c // vec) + 255) // 256)
            defines["LEGO_FILL_UNROLL"] = FILL_UNROLL
            reserved = runtime.FILL_FUSED                   # 16-byte windows on both sides
            detail += f", fill: affine {k}x+{c}, whole-sector windows"
        else:
            defines.update({"LEGO_FK": 0, "LEGO_FC": 0})
            reserved |= runtime.FILL_PASS
            detail += ", fill: vector fill pass + scatter"
    info = runtime.ProgramInfo(kind=runtime.KIND_SCATTER, elem_bytes=elem_bytes, n=n_src,
                               units=units, unit_threads=1, block=256, smem_bytes=0, reserved=reserved)
    src = _assemble(body, defines)
    return RemapPlan(runtime.KIND_SCATTER, n_dst, n_src, elem_bytes, False, False, src, info, detail)


def _remap_program(src_layout, dst_layout, elem_bytes, device: int, route=None, fill: bool = False):
    key = ("remap", _layout_key(src_layout), _layout_key(dst_layout), elem_bytes, fill,
           None if route is None else ("route", route.world, route.key), TRANSPOSE_VARIANT,
           BAND_ORDER, PERSIST_CTAS, TILE_ORDER, LOAD_HINT, STORE_HINT, TRANSPOSE_MINB,
           BAND_ROWS, BAND_DIAGS, BAND_WARPS, TRANSPOSE_WARPS, BOX_STAGING, NARROW, staging.BOX_TARGET, staging.BOX_STORE,
           staging.BOX_BULK, staging.BOX_THREADS)

    def build():
        plan = plan_remap(src_layout, dst_layout, elem_bytes, route, fill)
        # the sizes it was planned for travel with the program (set before publication)
        return plan.source, plan.info, {"n_dst": plan.n_dst, "n_src": plan.n_src, "kind": plan.kind,
                                        "gated": _needs_bijectivity_gate(src_layout, dst_layout, plan)}

    return _program(key, build, device)


def _map_program(layout, device: int):
    return _program(("map", _layout_key(layout)), lambda: index_map_source(layout), device)


# ---------------------------------------------------------------------------
# public operations
# ---------------------------------------------------------------------------

def _torch():
    import torch
    return torch


def _device(device):
    torch = _torch()
    if device is None:
        device = torch.device("cuda", torch.cuda.current_device())
    device = torch.device(device)
    if device.type != "cuda":
        raise ShapeMismatch(f"the backend runs on CUDA devices only, got {device}")
    if device.index is None:
        device = torch.device("cuda", torch.cuda.current_device())
    return device


def _check_out(out, shape, dtype, device, what, min_numel=None):
    """Caller-provided outputs go to the C ABI as bare pointers: check them."""
    if dtype is not None and out.dtype not in (dtype if isinstance(dtype, tuple) else (dtype,)):
        raise ShapeMismatch(f"{what}: out has dtype {out.dtype}, expected {dtype}")
    if out.device != device:
        raise ShapeMismatch(f"{what}: out is on {out.device}, expected {device}")
    if not out.is_contiguous():
        raise ShapeMismatch(f"{what}: out must be contiguous")
    if shape is not None and tuple(out.shape) != tuple(shape):
        raise ShapeMismatch(f"{what}: out has shape {tuple(out.shape)}, expected {tuple(shape)}")
    if min_numel is not None and out.numel() < min_numel:
        raise ShapeMismatch(f"{what}: out holds {out.numel()} elements, needs {min_numel}")


# reference validate() enumerates GenPs only up to this many points and
# "trusts" larger ones (pkg/src/lego/layout.py:718-719)
TRUST_BOUND = 4096
_BUILTIN_FACTORIES = ("identity_perm", "reverse_perm", "antidiag_perm")


def _builtin_genp(p) -> bool:
    """A GenP made by this package's built-in factories (bijective by
    construction); user GenPs -- even ones named like a built-in -- are not."""
    from . import layout as _layout
    fn = getattr(p.fwd, "concrete", None)
    return (getattr(fn, "__module__", None) == _layout.__name__
            and getattr(fn, "__qualname__", "").split(".")[0] in _BUILTIN_FACTORIES)


def _untrusted_genps(layout) -> bool:
    if layout is None:
        return False
    from .layout import GenP
    g = lower._group(layout)
    return any(isinstance(p, GenP) and p.size > TRUST_BOUND and not _builtin_genp(p)
               for stage in g.orders for p in stage.perms)


GENP_SAMPLES = 512          # points per user GenP checked before its first program


def check_genp_agreement(layout, samples: int = GENP_SAMPLES) -> None:
    """Every user GenP above the reference's trust bound must have a symbolic
    builder that agrees with its concrete callable: the device runs the
    symbolic form, the reference semantics is the concrete one
    (layout.py:187-200), and validate() only compares them up to 4096 points
    (layout.py:718-719).  Check ``samples`` deterministic points of each such
    GenP (forward and, when present, inverse) and raise ``LegoError`` on a
    disagreement, before any program is built from the layout."""
    from .expr import IntConst, eval_expr
    from .layout import GenP
    if layout is None:
        return
    g = lower._group(layout)
    for stage in g.orders:
        for p in stage.perms:
            if not (isinstance(p, GenP) and p.size > TRUST_BOUND and not _builtin_genp(p)):
                continue
            if _AGREED.get(id(p)) is p:
                continue
            n = p.size
            step = max(1, n // samples) | 1
            for k in range(min(samples, n)):
                f = (k * step + (k * 7919) % step) % n
                idx, rem = [], f
                for d in reversed(p.shape):
                    idx.append(rem % d)
                    rem //= d
                idx = tuple(reversed(idx))
                want = p.fwd.concrete(idx)
                got = eval_expr(as_expr_value(p.fwd.symbolic(tuple(IntConst(c) for c in idx))), {})
                if got != want:
                    raise LegoError(f"{p!r}: symbolic builder gives {got} at {idx}, the concrete function {want}; "
                                    "the device would evaluate the symbolic form")
                if p.inv_fn is not None:
                    wi = tuple(p.inv_fn.concrete(want))
                    gi = tuple(eval_expr(as_expr_value(e), {}) for e in p.inv_fn.symbolic(IntConst(want)))
                    if gi != wi:
                        raise LegoError(f"{p!r}: symbolic inverse gives {gi} at {want}, the concrete inverse {wi}")
            _AGREED[id(p)] = p                  # keeps p alive, so its id is not reused


_AGREED: dict = {}


def as_expr_value(e):
    from .expr import IntConst
    return e if not isinstance(e, int) else IntConst(e)


def _needs_bijectivity_gate(src_layout, dst_layout, plan):
    """Layouts to prove on the device before the first launch of a plan that
    *stores* through positions computed from a user GenP the reference only
    trusts (a non-injective GenP makes a scatter
    race).  Gathers enumerate the destination, so each element is written
    once whatever the map.  Returns [(layout, 'bijective'|'injective')]."""
    gates = []
    if plan.kind == runtime.KIND_SCATTER and _untrusted_genps(dst_layout):
        gates.append((dst_layout, "injective"))
    elif plan.kind == runtime.KIND_STAGED and plan.detail.startswith("source blocks"):
        gates += [(side, "bijective") for side in (src_layout, dst_layout) if _untrusted_genps(side)]
    elif plan.kind == runtime.KIND_BAND and plan.detail.endswith("scatter") and _untrusted_genps(dst_layout):
        gates.append((dst_layout, "bijective"))
    return gates


def _run_gates(prog, device):
    gates = getattr(prog, "gated", None)
    if not gates:
        return
    for layout, mode in gates:
        if mode == "injective":
            ok = check_injective(layout, device=device)
        else:
            ok = check_bijective(layout, device=device)
        if not ok:
            raise BijectivityViolation(f"layout {layout!r} is not {mode} on the device; a store through it "
                                       "would race (the reference only trusts GenPs above "
                                       f"{TRUST_BOUND} points)")
    prog.gated = []            # proven once per program


def apply_map(layout, *, dtype=None, device=None, first: int = 0, count: Optional[int] = None,
              out=None, stream=None):
    """``out[k] = layout.apply(canon_unflatten(dims, first + k))`` on the GPU
    (ExpandBy masked positions are -1)."""
    torch = _torch()
    n = lower.logical_size(layout)
    count = n - first if count is None else count
    if first < 0 or count < 0 or first + count > n:
        from .errors import OutOfBounds
        raise OutOfBounds(f"range [{first}, {first + count}) outside the logical space of {n}")
    dev = _device(out.device if out is not None else device)
    prog = _map_program(layout, dev.index)
    if out is None:
        dtype = dtype or (torch.int32 if lower.physical_size(layout) < 2 ** 31 else torch.int64)
        out = torch.empty(count, dtype=dtype, device=dev)
    else:
        _check_out(out, None, (torch.int32, torch.int64), dev, "apply_map", min_numel=count)
    with torch.cuda.device(dev):
        runtime.check(runtime.lib().lego_apply_map(prog.handle, out.data_ptr(), out.element_size(),
                                                   first, count, runtime.stream_handle(stream)),
                      "lego_apply_map")
    LAUNCHES[0] += 1
    return out


def inv_map(layout, *, dtype=None, device=None, first: int = 0, count: Optional[int] = None,
            out=None, stream=None):
    """``out[k] = canon_flatten(dims, layout.inv(first + k))`` on the GPU.
    Injective-mode layouts export ``apply`` only and raise, as the reference's
    ``GroupBy.inv`` does (layout.py:321-322)."""
    torch = _torch()
    if getattr(lower._group(layout), "injective", False):
        from .errors import LegoError
        raise LegoError("injective layout exports apply only, not inv")
    n = lower.physical_size(layout)
    count = n - first if count is None else count
    if first < 0 or count < 0 or first + count > n:
        from .errors import OutOfBounds
        raise OutOfBounds(f"range [{first}, {first + count}) outside the physical space of {n}")
    dev = _device(out.device if out is not None else device)
    prog = _map_program(layout, dev.index)
    if out is None:
        dtype = dtype or (torch.int32 if lower.logical_size(layout) < 2 ** 31 else torch.int64)
        out = torch.empty(count, dtype=dtype, device=dev)
    else:
        _check_out(out, None, (torch.int32, torch.int64), dev, "inv_map", min_numel=count)
    with torch.cuda.device(dev):
        runtime.check(runtime.lib().lego_inv_map(prog.handle, out.data_ptr(), out.element_size(),
                                                 first, count, runtime.stream_handle(stream)),
                      "lego_inv_map")
    LAUNCHES[0] += 1
    return out


def _check_hits(layout, fn_name, device, stream):
    torch = _torch()
    dev = _device(device)
    prog = _map_program(layout, dev.index)
    hist = torch.empty(prog.info.units, dtype=torch.int32, device=dev)
    bad = runtime.I64()
    with torch.cuda.device(dev):
        runtime.check(getattr(runtime.lib(), fn_name)(prog.handle, hist.data_ptr(), ctypes.byref(bad),
                                                      runtime.stream_handle(stream)), fn_name)
    LAUNCHES[0] += 2
    return bad.value


def check_bijective(layout, *, device=None, stream=None, raise_on_failure: bool = False) -> bool:
    """Device-side proof that ``apply`` hits every position exactly once."""
    bad = _check_hits(layout, "lego_check_bijective", device, stream)
    if bad and raise_on_failure:
        raise BijectivityViolation(f"{bad} positions are not hit exactly once")
    return bad == 0


def check_injective(layout, *, device=None, stream=None, raise_on_failure: bool = False) -> bool:
    """Device-side proof that ``apply`` hits no position twice (injective-mode
    layouts may leave positions unhit)."""
    bad = _check_hits(layout, "lego_check_injective", device, stream)
    if bad and raise_on_failure:
        raise BijectivityViolation(f"{bad} positions are hit more than once")
    return bad == 0


def remap_plan(src_layout, dst_layout, elem_bytes: int) -> RemapPlan:
    """The lowering decision (kernel family, geometry) without compiling."""
    return plan_remap(src_layout, dst_layout, elem_bytes)


def remap(src, src_layout=None, dst_layout=None, *, out=None, fill=None, stream=None):
    """Move ``src`` (shape ``(..., n_src)``) into the destination layout:
    for every logical index x, ``out[..., dst.apply(x)] = src[..., src.apply(x)]``.
    ``None`` on either side means row-major over the other side's dims.

    Injective-mode destinations (no inverse) leave positions no x hits:
    with ``out`` given and ``fill=None`` they keep ``out``'s values;
    otherwise they are set to ``fill`` (default 0 for a fresh output) by the
    same launch.  Other layouts write every position; ``fill`` is unused."""
    torch = _torch()
    if not src.is_cuda:
        raise ShapeMismatch("remap takes a CUDA tensor (no CPU path)")
    elem = src.element_size()
    lower.check_pair(src_layout, dst_layout)
    dev = src.device
    injective = dst_layout is not None and getattr(lower._group(dst_layout), "injective", False)
    want_fill = injective and src_layout is None and (fill is not None or out is None)
    prog = _remap_program(src_layout, dst_layout, elem, dev.index, fill=want_fill)
    f_dst, n_src = prog.n_dst, prog.n_src
    if src.numel() % n_src:
        raise ShapeMismatch(f"source of {src.numel()} elements is not a batch of layouts of "
                            f"size {n_src}")
    src = src.contiguous()
    batch = src.numel() // n_src
    batch_shape = tuple(src.shape[:-1]) if src.dim() and src.shape[-1] == n_src else (batch,)
    if out is None:
        out = torch.empty(*batch_shape, f_dst, dtype=src.dtype, device=dev)
    else:
        _check_out(out, None, src.dtype, dev, "remap", min_numel=batch * f_dst)
    if batch == 0:
        return out
    _run_gates(prog, dev)
    fill_buf = None
    if want_fill:
        fill_buf = torch.tensor([fill if fill is not None else 0], dtype=src.dtype).view(torch.uint8).numpy()
        fill_buf = ctypes.create_string_buffer(fill_buf.tobytes(), elem)
    with torch.cuda.device(dev):
        st = runtime.stream_handle(stream)
        done = 0
        while done < batch:
            b = min(65535, batch - done)
            s_ptr, d_ptr = src.data_ptr() + done * n_src * elem, out.data_ptr() + done * f_dst * elem
            if fill_buf is not None:
                runtime.check(runtime.lib().lego_remap_fill(prog.handle, s_ptr, d_ptr, b, n_src, f_dst, fill_buf, st),
                              "lego_remap_fill")
                LAUNCHES[0] += 1 if prog.info.reserved & runtime.FILL_FUSED else 2
            else:
                runtime.check(runtime.lib().lego_remap(prog.handle, s_ptr, d_ptr, b, n_src, f_dst, st),
                              "lego_remap")
                LAUNCHES[0] += 1
            done += b
    return out


def remap_routed(src, src_layout, dst_layout, peers, route: Route, *, stream=None):
    """One remap whose destination is spread over ``route.world`` buffers:
    destination element v lands in buffer ``route.peer(v)`` at element offset
    ``route.off(v)``.  ``peers`` is an int64 CUDA tensor holding the buffers'
    device addresses -- for a cross-rank exchange, the NVLink-mapped
    symmetric buffers of every rank, so the remap and the all-to-all are one
    kernel (``shard.transpose_rows_fused``).  One matrix per call; the caller
    orders the peers' reads after the stores (a barrier)."""
    torch = _torch()
    if not src.is_cuda or not peers.is_cuda or peers.dtype != torch.int64:
        raise ShapeMismatch("remap_routed takes a CUDA source and an int64 CUDA peer table")
    if peers.numel() != route.world:
        raise ShapeMismatch(f"peer table has {peers.numel()} entries for {route.world} peers")
    if peers.device != src.device:
        raise ShapeMismatch("the peer table must live on the source's device")
    elem = src.element_size()
    lower.check_pair(src_layout, dst_layout)
    dev = src.device
    prog = _remap_program(src_layout, dst_layout, elem, dev.index, route)
    if src.numel() != prog.n_src:
        raise ShapeMismatch(f"routed remap moves one layout of {prog.n_src} elements, got {src.numel()}")
    src = src.contiguous()
    with torch.cuda.device(dev):
        runtime.check(runtime.lib().lego_remap(prog.handle, src.data_ptr(), peers.data_ptr(), 1,
                                               prog.n_src, prog.n_dst, runtime.stream_handle(stream)),
                      "lego_remap")
    LAUNCHES[0] += 1


def gather(src, layout, **kw):
    """Physical buffer in ``layout`` -> logical row-major order."""
    return remap(src, layout, None, **kw)


def scatter(src, layout, **kw):
    """Logical row-major data -> physical buffer in ``layout``."""
    return remap(src, None, layout, **kw)


# ---------------------------------------------------------------------------
# fixed kernels
# ---------------------------------------------------------------------------

SOFTMAX_THREADS = 256          # T of the thread layout (softmax_kernels.cuh kThreads)
SOFTMAX_MAX_ITS = 16           # float4 vectors per thread held in registers


def softmax_layout(cols: int, rows: Optional[int] = None):
    """The softmax thread/data layout of the paper:
    ``GroupBy([rows], [cols/(4T)], [T], [4]).OrderBy(Row(rows, cols))`` --
    element (row, it, tid, v) of the thread decomposition lives at its
    ``apply``.  ``rows`` defaults to the largest row count a program serves
    (2^36 elements), so one program covers every batch of rows."""
    from .layout import GroupBy, row
    t4 = 4 * SOFTMAX_THREADS
    if cols % t4:
        raise ShapeMismatch(f"the register softmax layout needs cols % {t4} == 0, got {cols}")
    rows = rows if rows is not None else max(1, (1 << 36) // cols)
    return GroupBy([rows], [cols // t4], [SOFTMAX_THREADS], [4]).order_by(row(rows, cols))


def softmax_source(cols: int):
    """NVRTC source of the register softmax with its offsets generated from
    :func:`softmax_layout` (gen::vec_of = apply(row, it, tid, 0) / 4)."""
    lay = softmax_layout(cols)
    rows = lay.dims[0]
    its = cols // (4 * SOFTMAX_THREADS)
    r = Var("row", VarRange(0, rows))
    it = Var("it", VarRange(0, its))
    tid = Var("tid", VarRange(0, SOFTMAX_THREADS))
    pos = lower.apply_flat(lay, lower.as_expr(((r * its + it) * SOFTMAX_THREADS + tid) * 4))
    vec = lower.simplify(lower.as_expr(lower.simplify(lower.as_expr(pos)) // 4))
    body = codegen.constant("COLS", cols) + codegen.constant("ITS", its)
    body += codegen.generate("vec_of", [r, it, tid], {"k": vec}).source
    src = ("#define SM_GEN 1\n" + _text("lego_index.cuh").replace("#pragma once", "") + "\nnamespace gen {\n"
           + body + "}\n" + _text("softmax_kernels.cuh").replace("#pragma once", ""))
    info = runtime.ProgramInfo(kind=runtime.KIND_SOFTMAX, elem_bytes=4, n=cols, units=rows, unit_threads=1,
                               block=SOFTMAX_THREADS, smem_bytes=0)
    return src, info


def softmax_program(cols: int, device=None):
    dev = _device(device)
    return _program(("softmax", cols), lambda: softmax_source(cols), dev.index)


def softmax_generated(cols: int) -> bool:
    """Whether rows of this length take the LEGO-generated program."""
    t4 = 4 * SOFTMAX_THREADS
    return cols > 0 and cols % t4 == 0 and cols // t4 <= SOFTMAX_MAX_ITS


def softmax(x, *, out=None, stream=None):
    """Row softmax over the last dim of a contiguous fp32 CUDA tensor.  Rows
    of a whole number of 4T-float passes (up to 16) run the program generated
    from :func:`softmax_layout`; other lengths the library's built-in kernels."""
    torch = _torch()
    if x.dtype != torch.float32 or not x.is_cuda or x.dim() == 0:
        raise ShapeMismatch("softmax takes a CUDA float32 tensor")
    x = x.contiguous()
    cols = x.shape[-1]
    rows = x.numel() // cols if cols else 0
    if out is None:
        out = torch.empty_like(x)
    else:
        _check_out(out, tuple(x.shape), torch.float32, x.device, "softmax")
    if x.numel() == 0:
        return out
    with torch.cuda.device(x.device):
        st = runtime.stream_handle(stream)
        aligned = (x.data_ptr() | out.data_ptr()) % 16 == 0
        if rows and softmax_generated(cols) and aligned and rows <= (1 << 36) // cols:
            prog = softmax_program(cols, x.device)
            runtime.check(runtime.lib().lego_softmax_run(prog.handle, x.data_ptr(), out.data_ptr(), rows, cols,
                                                         st), "lego_softmax_run")
        else:
            runtime.check(runtime.lib().lego_softmax_f32(x.data_ptr(), out.data_ptr(), rows, cols, st),
                          "lego_softmax_f32")
    LAUNCHES[0] += 1
    return out


def nw_score(sim, penalty: int, *, layout=None, out=None, stream=None):
    """Needleman-Wunsch score matrices for int32 similarity ``(..., n, n)``.

    ``layout`` is a LEGO layout of the n x n cell grid (:func:`.nw.nw_layout`)
    whose tile order and shared-memory cell order drive the wavefront kernel
    (:mod:`.nw`); ``None`` runs the library's built-in instance of the default
    layout (128-column strips)."""
    torch = _torch()
    if sim.dtype != torch.int32 or not sim.is_cuda or sim.dim() < 2 or sim.shape[-1] != sim.shape[-2]:
        raise ShapeMismatch("nw_score takes a CUDA int32 tensor of shape (..., n, n)")
    sim = sim.contiguous()
    n = sim.shape[-1]
    batch = 1
    for d in sim.shape[:-2]:
        batch *= d
    shape = (*sim.shape[:-2], n + 1, n + 1)
    if out is None:
        out = torch.empty(*shape, dtype=torch.int32, device=sim.device)
    else:
        _check_out(out, shape, torch.int32, sim.device, "nw_score")
    with torch.cuda.device(sim.device):
        st = runtime.stream_handle(stream)
        if layout is None or n == 0 or batch == 0:
            runtime.check(runtime.lib().lego_nw_i32(sim.data_ptr(), out.data_ptr(), n, int(penalty), batch, st),
                          "lego_nw_i32")
        else:
            from . import nw
            prog = nw.nw_program(layout, n, device=sim.device)
            if not nw.needs_program(prog.defines):
                # the layout lowers to no generated map (row-major strips, row-major
                # ring): the library's nvcc-built instance of the same template
                runtime.check(runtime.lib().lego_nw_i32(sim.data_ptr(), out.data_ptr(), n, int(penalty), batch,
                                                        st), "lego_nw_i32")
            else:
                runtime.check(runtime.lib().lego_nw_run(prog.handle, sim.data_ptr(), out.data_ptr(), n,
                                                        int(penalty), batch, st), "lego_nw_run")
    LAUNCHES[0] += 2
    return out


NW_EMPTY_WORD = -2139062144        # 0x80808080: the sentinel of not-yet-published NW edge words


def nw_band_words(n: int, strips: int, batch: int = 1) -> int:
    """int32 words of a band's edge columns (``bnd`` of :func:`nw_score_band`)."""
    return batch * strips * (-(-n // 32) * 32)


def nw_score_band(sim, penalty: int, strips, bnd, *, left=None, left_strips: int = 0, out=None,
                  max_ctas: int = 0, stream=None):
    """Strips ``strips = (begin, end)`` (128 columns each) of the NW score of
    ``sim`` into ``out`` (full (..., n+1, n+1) size; only those columns and the
    borders are written).  ``bnd`` (int32, :func:`nw_band_words` words, preset
    to :data:`NW_EMPTY_WORD` before any reader starts) receives the band's edge
    columns (batch x strips x n_pad, n_pad = n rounded up to 32); ``left`` is
    the previous band's ``bnd`` tensor with ``left_strips`` strips, possibly a
    peer GPU's symmetric-memory buffer: its last strip's column is read
    (``None`` when ``begin == 0``).  The multi-GPU building block of
    :func:`.shard.nw_score_banded`."""
    torch = _torch()
    if sim.dtype != torch.int32 or not sim.is_cuda or sim.dim() < 2 or sim.shape[-1] != sim.shape[-2]:
        raise ShapeMismatch("nw_score_band takes a CUDA int32 tensor of shape (..., n, n)")
    sim = sim.contiguous()
    n = sim.shape[-1]
    batch = 1
    for d in sim.shape[:-2]:
        batch *= d
    begin, end = (int(x) for x in strips)
    shape = (*sim.shape[:-2], n + 1, n + 1)
    if out is None:
        out = torch.empty(*shape, dtype=torch.int32, device=sim.device)
    else:
        _check_out(out, shape, torch.int32, sim.device, "nw_score_band")
    if bnd.dtype != torch.int32 or bnd.device != sim.device or bnd.numel() < nw_band_words(n, end - begin, batch):
        raise ShapeMismatch("bnd must be int32 on sim's device with nw_band_words(n, strips, batch) words")
    left_ptr, left_stride = None, 0
    if left is not None:
        n_pad = -(-n // 32) * 32
        if left_strips < 1 or left.numel() < nw_band_words(n, left_strips, batch):
            raise ShapeMismatch("left must hold the previous band's left_strips edge columns per matrix")
        left_ptr = left.data_ptr() + 4 * (left_strips - 1) * n_pad     # its last strip
        left_stride = left_strips * n_pad
    with torch.cuda.device(sim.device):
        st = runtime.stream_handle(stream)
        runtime.check(runtime.lib().lego_nw_band_i32(sim.data_ptr(), out.data_ptr(), n, int(penalty), batch, begin,
                                                     end, bnd.data_ptr(), left_ptr, int(left_stride),
                                                     int(max_ctas), st), "lego_nw_band_i32")
    LAUNCHES[0] += 2
    return out


# measured (scripts/ab_gemm_group.py, 8192^3, 4 alternating runs each): G = 32 685 us,
# 24 688, 48 688, 16 692, 64 695
GEMM_RASTER_GROUP = int(os.environ.get("LEGO_GEMM_GROUP", "32"))


def gemm(a, b, *, out=None, raster: Optional[int] = None, a_col: bool = False, b_col: bool = False,
         stream=None):
    """``C = A @ B.T`` for bf16 ``A (..., M, K)`` and ``B (..., N, K)`` on tcgen05.

    ``a_col`` / ``b_col``: the operand is passed MN-major instead, ``a`` as
    ``(..., K, M)`` (A = a^T) and ``b`` as ``(..., K, N)`` (B = b^T) -- the
    Row/Col operand data layouts of the paper's matmul variants, consumed
    directly as MN-major UMMA operands.  ``raster`` = G selects the LEGO tile
    raster ``GroupBy([MB/G, NB, G]).OrderBy(Row(MB/G, NB, G))`` (0 = row-major)."""
    if raster is None:
        raster = GEMM_RASTER_GROUP
    torch = _torch()
    if a.dtype != torch.bfloat16 or b.dtype != torch.bfloat16 or not a.is_cuda or not b.is_cuda:
        raise ShapeMismatch("gemm takes CUDA bfloat16 tensors")
    if a.device != b.device:
        raise ShapeMismatch(f"gemm operands on different devices: {a.device} and {b.device}")
    if a.dim() < 2 or b.dim() < 2 or tuple(a.shape[:-2]) != tuple(b.shape[:-2]):
        raise ShapeMismatch(f"gemm needs matching batch dims: {tuple(a.shape)} vs {tuple(b.shape)}")
    a, b = a.contiguous(), b.contiguous()
    K, M = (a.shape[-2], a.shape[-1]) if a_col else (a.shape[-1], a.shape[-2])
    Kb, N = (b.shape[-2], b.shape[-1]) if b_col else (b.shape[-1], b.shape[-2])
    if Kb != K:
        raise ShapeMismatch(f"inner dims differ: {K} vs {Kb}")
    batch = 1
    for d in a.shape[:-2]:
        batch *= d
    if out is None:
        out = torch.empty(*a.shape[:-2], M, N, dtype=torch.bfloat16, device=a.device)
    else:
        _check_out(out, (*a.shape[:-2], M, N), torch.bfloat16, a.device, "gemm")
    if batch == 0 or M == 0 or N == 0:
        return out
    if K == 0:
        return out.zero_()
    with torch.cuda.device(a.device):
        runtime.check(runtime.lib().lego_gemm_bf16_ex(a.data_ptr(), b.data_ptr(), out.data_ptr(), M, N, K,
                                                      batch, raster, int(a_col), int(b_col),
                                                      runtime.stream_handle(stream)),
                      "lego_gemm_bf16_ex")
    LAUNCHES[0] += 1
    return out


def compile_template(template_text: str, manifest_text: str, layouts=None) -> "runtime.Module":
    """Instantiate a LEGO ``.cu`` template (reference ``template.instantiate``,
    template.py:522-537) with the ``cuda`` target profile, compile it for
    sm_100a (NVRTC, cubin cached on disk) and load it: the paper's CUDA
    integration route.  The manifest must select
    ``[target] cuda``; the index helpers (floor div/mod, exact isqrt) are
    prepended."""
    from . import template as T
    manifest = T.parse_manifest(manifest_text)
    src = T.instantiate(T.parse_template(template_text), manifest, layouts=layouts)
    return runtime.Module(runtime.compile_cubin(_text("lego_index.cuh") + "\n" + src))


def gemm_raster(mtiles: int, ntiles: int, batch: int = 1, group: Optional[int] = None, *, device=None):
    """The GEMM kernels' tile order as the device evaluates it: row t of the
    (mtiles*ntiles*batch, 3) int32 result is (batch, m-block, n-block) of
    tile t.  ``group`` = G of the grouped raster (0 = row-major)."""
    torch = _torch()
    group = GEMM_RASTER_GROUP if group is None else group
    dev = _device(device)
    out = torch.empty(mtiles * ntiles * batch, 3, dtype=torch.int32, device=dev)
    with torch.cuda.device(dev):
        runtime.check(runtime.lib().lego_gemm_raster(out.data_ptr(), mtiles, ntiles, batch, group,
                                                     runtime.stream_handle(None)), "lego_gemm_raster")
    LAUNCHES[0] += 1
    return out


def matmul(a, b, *, a_layout="row", b_layout="row", out=None, **kw):
    """``C = A @ B`` with ``A`` (M x K) and ``B`` (K x N) given in the Row or Col
    data layout of the paper's four matmul variants: a
    Row operand is stored row-major, a Col operand column-major (i.e. the
    tensor passed holds its transpose, ``A^T`` as (..., K, M) / ``B^T`` as
    (..., N, K)).  Every variant runs as one tcgen05 GEMM; nothing is
    transposed in memory.

    ``a_layout`` / ``b_layout`` may also be LEGO data layouts over the
    logical (M, K) / (K, N) operand (the reference matmul workflow's
    ``Data`` layouts, test_acceptance.py:211-234), e.g.
    ``GroupBy([M,K]).OrderBy(Row(M,K))`` or ``...OrderBy(Col(K,M))``; their
    affine strides (:func:`.gemm_layouts.operand_strides`) select the TMA
    operand major, and the tensor passed is the layout's physical buffer."""
    from . import gemm_layouts as GL
    if not isinstance(a_layout, str):
        M, K = a_layout.dims
        maj = GL.operand_major(a_layout, "A")
        if a.numel() != M * K:
            raise ShapeMismatch(f"A holds {a.numel()} elements, its layout {M * K}")
        a = a.reshape((M, K) if maj == "row" else (K, M))
        a_layout = maj
    if not isinstance(b_layout, str):
        Kb, N = b_layout.dims
        maj = GL.operand_major(b_layout, "B")
        if b.numel() != Kb * N:
            raise ShapeMismatch(f"B holds {b.numel()} elements, its layout {Kb * N}")
        b = b.reshape((Kb, N) if maj == "row" else (N, Kb))
        b_layout = maj
    if a_layout not in ("row", "col") or b_layout not in ("row", "col"):
        raise ShapeMismatch("a_layout / b_layout must be 'row', 'col' or a 2-D LEGO layout")
    # gemm computes A @ B'^T with B' = B^T given K-major (N x K) or MN-major (K x N)
    return gemm(a, b, out=out, a_col=a_layout == "col", b_col=b_layout == "row", **kw)
