"""Needleman-Wunsch wavefront driven by a LEGO layout (BASELINE.json config 4b).

The paper's NW kernel takes its irregular anti-diagonal indexing from LEGO
(``PAPER.md:1298-1301``; the layout of its Eq. (layout-fig6),
``PAPER.md:702-708``).  Here the user describes the cell grid of an
``n x n`` alignment with a LEGO layout, and the layout is lowered into the
wavefront kernel (``csrc/nw_kernels.cuh``):

``GroupBy([NR*H, NC*128]).OrderBy(RegP([NR, H, NC, 128], [1, 3, 2, 4])).OrderBy(T, I)``

i.e. ``position(a*H + r, b*128 + c) = T(a, b) * (H*128) + I(r, c)``
(reference semantics: ``GroupBy.apply``, ``pkg/src/lego/layout.py:313-318``;
mixed-radix ``OrderBy``, ``layout.py:237-258``).  The grid is the alignment
padded to whole tiles (``NR = ceil(n/H)``, ``NC = ceil(n/128)``).

* ``T`` -- any LEGO permutation of the ``NR x NC`` tile grid (``RegP``,
  built-in or user ``GenP``) -- is the **tile order**: CTAs claim tiles from
  an atomic ticket and ticket ``t`` is tile ``T^-1(t)`` (generated as
  ``gen::tile_of`` from the layout's symbolic inverse).  A tile can only run
  after its upper and left neighbours, so ``T`` must be a topological order
  of that dependency graph; :func:`nw_program` proves it exhaustively (on the
  device through the generated map, and with the layout's own concrete
  callables on the host) and raises :class:`~.errors.UnsupportedNode`
  otherwise.  Any such order is deadlock-free on a persistent grid: every
  tile a claimed tile waits on was claimed earlier by a running CTA.
* ``I`` -- a permutation of a tile's ``H x 128`` cells -- is the
  **shared-memory cell order** of the tile in the kernel's staging ring (the
  paper permutes NW's shared buffer with LEGO's anti-diagonal layout to
  avoid bank conflicts).  The ring streams rows and every lane moves one
  16-byte group of 4 columns, so ``I`` must map each row onto itself and
  each aligned 4-column group onto an aligned contiguous group (e.g. an XOR
  or rotation swizzle of the 32 lane groups); proven exhaustively the same
  way.  ``gen::slot(r, g)`` is generated from it.

``H = n`` (one tile row: column strips) is the library's built-in default
layout (``lego_nw_i32``); every other layout is compiled by NVRTC into its
own program (``lego_nw_run``).  Results never depend on the layout -- it
changes only the execution order and data placement -- so every layout is
checked bit-exact against the same CPU DP (``tests/test_nw_layouts.py``).
"""

from __future__ import annotations

from typing import Optional, Tuple

from . import codegen, lower, runtime
from .errors import ShapeMismatch, UnsupportedNode
from .expr import IntConst, Var, VarRange
from .layout import GenP, GroupBy, OrderBy, RegP, resolve_builtin_perm

STRIP = 128                       # columns per tile (32 lanes x 4 columns)
LANES = 32
BLK = 32                          # rows per staging block
# nw_kernels.cuh SMEM_BYTES: 256-row ring (8 blocks) + boundary ring + mbarriers + control + top row
NSLOT = 8


def smem_bytes(nslot: int = NSLOT, bnd_rows: int = 256) -> int:
    return nslot * 32 * STRIP * 4 + bnd_rows * 4 + nslot * 8 + 64 + (STRIP + 4) * 4


SMEM_BYTES = smem_bytes()
KIND_NW = 6


def _grid(n: int, tile_rows: Optional[int]) -> Tuple[int, int, int]:
    h = max(n, 1) if tile_rows is None else int(tile_rows)
    if h < 1:
        raise ShapeMismatch("tile_rows must be positive")
    nr = max(1, -(-n // h))
    nc = max(1, -(-n // STRIP))
    return h, nr, nc


def _perm_for(spec, shape, what: str):
    """A permutation over `shape` from a name ('row', 'col', a registered
    built-in such as 'antidiag'), a RegP/GenP, or a sequence of them."""
    if spec is None or spec == "row":
        return (RegP(shape, list(range(1, len(shape) + 1))),)
    if spec == "col":
        return (RegP(shape, list(range(len(shape), 0, -1))),)
    if isinstance(spec, str):
        return (resolve_builtin_perm(spec, shape),)
    if isinstance(spec, (RegP, GenP)):
        perms = (spec,)
    else:
        perms = tuple(spec)
    dims = tuple(d for p in perms for d in p.dims)
    if dims != tuple(shape):
        raise ShapeMismatch(f"{what} covers dims {dims}, expected {tuple(shape)}")
    return perms


def nw_layout(n: int, tile_rows: Optional[int] = None, tile_order=None, cell_order=None) -> GroupBy:
    """The LEGO layout of an n x n NW cell grid for :func:`kernels.nw_score`.

    ``tile_rows`` = H (default n: 128-column strips); ``tile_order`` = T over
    the (ceil(n/H), ceil(n/128)) tile grid ('row' default, 'col',
    'antidiag', or any RegP/GenP); ``cell_order`` = I over (H, 128)."""
    h, nr, nc = _grid(n, tile_rows)
    split = OrderBy(RegP([nr, h, nc, STRIP], [1, 3, 2, 4]))
    if tile_order is None and cell_order is None:
        return GroupBy([nr * h, nc * STRIP], orders=(split,))
    t = _perm_for(tile_order, (nr, nc), "tile_order")
    i = _perm_for(cell_order, (h, STRIP), "cell_order")
    return GroupBy([nr * h, nc * STRIP], orders=(split, OrderBy(*t, *i)))


class NwParts:
    """The pieces of an NW layout the kernel consumes."""

    def __init__(self, n, h, nr, nc, tiles: GroupBy, cells: GroupBy):
        self.n, self.h, self.nr, self.nc = n, h, nr, nc
        self.tiles, self.cells = tiles, cells

    def __repr__(self):
        return f"NwParts(n={self.n}, tile {self.h}x{STRIP}, grid {self.nr}x{self.nc})"


_FORM = ("GroupBy([NR*H, NC*128]).OrderBy(RegP([NR,H,NC,128],[1,3,2,4])).OrderBy(T, I) "
         "with T over [NR,NC] and I over [H,128], NR = ceil(n/H), NC = ceil(n/128)")


def nw_parts(layout, n: int) -> NwParts:
    """Split a layout of the NW cell grid into tile order and cell order
    (raises UnsupportedNode for layouts of another form)."""
    if not isinstance(layout, GroupBy) or layout.injective:
        raise UnsupportedNode(f"NW layouts must be {_FORM}")
    layout._check()
    if len(layout.dims) != 2 or not 1 <= len(layout.orders) <= 2:
        raise UnsupportedNode(f"NW layouts must be {_FORM}")
    first = layout.orders[0].perms
    if len(first) != 1 or not isinstance(first[0], RegP) or first[0].sigma != (1, 3, 2, 4) \
            or len(first[0].shape) != 4:
        raise UnsupportedNode(f"the first stage must split the grid into tiles: {_FORM}")
    nr, h, nc, w = first[0].shape
    if w != STRIP:
        raise UnsupportedNode(f"NW tiles are {STRIP} columns wide (one warp x 4 columns), got {w}")
    if tuple(layout.dims) != (nr * h, nc * STRIP):
        raise UnsupportedNode(f"NW layouts must be {_FORM}")
    if n == 0:
        raise ShapeMismatch("an empty alignment has no cell layout")
    if nr != -(-n // h) or nc != -(-n // STRIP):
        raise ShapeMismatch(f"layout grid {nr}x{nc} of {h}x{STRIP} tiles does not cover n = {n} exactly "
                            f"(need {-(-n // h)}x{-(-n // STRIP)})")
    if nr > 1 and h % BLK:
        raise UnsupportedNode(f"tile rows must be a multiple of {BLK} when there is more than one tile row")
    if len(layout.orders) == 1:
        t = (RegP([nr, nc], [1, 2]),)
        i = (RegP([h, STRIP], [1, 2]),)
    else:
        perms = layout.orders[1].perms
        acc, k = (), 0
        while k < len(perms) and len(acc) < 2:
            acc += tuple(perms[k].dims)
            k += 1
        if acc != (nr, nc) or tuple(d for p in perms[k:] for d in p.dims) != (h, STRIP):
            raise UnsupportedNode(f"the second stage must be (T over [{nr},{nc}], I over [{h},{STRIP}]): {_FORM}")
        t, i = perms[:k], perms[k:]
    return NwParts(n, h, nr, nc, GroupBy([nr, nc], orders=(OrderBy(*t),)),
                   GroupBy([h, STRIP], orders=(OrderBy(*i),)))


# ---------------------------------------------------------------------------
# proofs (exhaustive; device through the generated maps, host through the
# layout's own concrete callables -- the reference semantics, layout.py:187-200)
# ---------------------------------------------------------------------------

HOST_CHECK_LIMIT = 1 << 14        # tiles / rows checked with the concrete callables in full
HOST_SAMPLE = 4096                # otherwise this many, spread over the space


def _host_points(total: int):
    if total <= HOST_CHECK_LIMIT:
        return range(total)
    step = max(1, total // HOST_SAMPLE)
    return range(0, total, step)


def host_check_tile_order(parts: NwParts) -> None:
    """The tile-order proof with the layout's concrete callables (reference
    ``GroupBy.apply`` semantics): exhaustive up to HOST_CHECK_LIMIT tiles,
    else the neighbour relations of a spread sample of tiles."""
    nr, nc = parts.nr, parts.nc
    ap = parts.tiles.apply
    exhaustive = nr * nc <= HOST_CHECK_LIMIT
    seen = set()
    for x in _host_points(nr * nc):
        a, b = divmod(x, nc)
        p = ap((a, b))
        if not 0 <= p < nr * nc:
            raise UnsupportedNode(f"tile order maps tile ({a}, {b}) outside the grid ({p})")
        if exhaustive:
            if p in seen:
                raise UnsupportedNode("tile order is not a permutation of the tile grid")
            seen.add(p)
        if a > 0 and ap((a - 1, b)) >= p:
            raise UnsupportedNode(f"tile order puts tile ({a}, {b}) before its upper neighbour ({a - 1}, {b}); "
                                  "the wavefront needs a topological order")
        if b > 0 and ap((a, b - 1)) >= p:
            raise UnsupportedNode(f"tile order puts tile ({a}, {b}) before its left neighbour ({a}, {b - 1}); "
                                  "the wavefront needs a topological order")


def check_tile_order(parts: NwParts, device=None) -> None:
    """T is a bijection of the tile grid and every tile comes after its upper
    and left neighbours (so also after its diagonal one): on the host with
    the concrete callables, then exhaustively on the device through the
    generated maps the kernel runs (which must agree with the host)."""
    import torch

    from . import kernels as K
    nr, nc = parts.nr, parts.nc
    if nr * nc == 1:
        return
    host_check_tile_order(parts)
    pos = K.apply_map(parts.tiles, dtype=torch.int64, device=device)
    inv = K.inv_map(parts.tiles, dtype=torch.int64, device=device)
    ar = torch.arange(nr * nc, device=pos.device)
    if not torch.equal(torch.sort(pos).values, ar):
        raise UnsupportedNode("tile order is not a permutation of the tile grid")
    if not torch.equal(inv[pos], ar):
        raise UnsupportedNode("tile order: the generated inverse disagrees with apply")
    grid = pos.view(nr, nc)
    if nr > 1 and not bool((grid[1:] > grid[:-1]).all()):
        a, b = [int(v) for v in torch.nonzero(grid[1:] <= grid[:-1])[0]]
        raise UnsupportedNode(f"tile order puts tile ({a + 1}, {b}) before its upper neighbour ({a}, {b}); "
                              "the wavefront needs a topological order")
    if nc > 1 and not bool((grid[:, 1:] > grid[:, :-1]).all()):
        a, b = [int(v) for v in torch.nonzero(grid[:, 1:] <= grid[:, :-1])[0]]
        raise UnsupportedNode(f"tile order puts tile ({a}, {b + 1}) before its left neighbour ({a}, {b}); "
                              "the wavefront needs a topological order")
    host = pos.cpu().tolist()
    for x in _host_points(nr * nc):
        a, b = divmod(x, nc)
        if parts.tiles.apply((a, b)) != host[x]:
            raise UnsupportedNode(f"tile order: concrete apply({a}, {b}) != generated {host[x]} "
                                  "(symbolic and concrete functions of a GenP disagree)")


def host_check_cell_order(parts: NwParts) -> None:
    """The cell-order conditions with the concrete callables (exhaustive up
    to HOST_CHECK_LIMIT rows x 128, else a spread sample of rows)."""
    h = parts.h
    ap = parts.cells.apply
    rows = range(h) if h * STRIP <= HOST_CHECK_LIMIT * 8 else range(0, h, max(1, h // 64))
    for r in rows:
        slots = set()
        for g in range(LANES):
            base = ap((r, 4 * g))
            if base // STRIP != r or base % 4:
                raise UnsupportedNode(f"cell order must keep tile row {r} in its ring row with aligned "
                                      f"4-column groups (group {g} -> {base})")
            for k in range(1, 4):
                if ap((r, 4 * g + k)) != base + k:
                    raise UnsupportedNode("cell order must move each lane's 4-column group as one "
                                          "contiguous 16-byte group")
            slots.add((base % STRIP) // 4)
        if len(slots) != LANES:
            raise UnsupportedNode(f"cell order is not a permutation of row {r}'s lane groups")


def slot_identity(parts: NwParts) -> bool:
    r = Var("r", VarRange(0, parts.h))
    g = Var("g", VarRange(0, LANES))
    return lower.simplify(_slot_expr(parts, r, g) - g) == IntConst(0)


def _slot_expr(parts: NwParts, r: Var, g: Var):
    pos = lower.apply_flat(parts.cells, lower.as_expr(r * STRIP + g * 4))
    return lower.simplify(lower.as_expr((pos - r * STRIP) // 4))


def check_cell_order(parts: NwParts, device=None) -> None:
    """I maps every tile row onto itself and every aligned 4-column group onto
    an aligned contiguous group (one 16-byte ring slot)."""
    import torch

    from . import kernels as K
    h = parts.h
    host_check_cell_order(parts)
    pos = K.apply_map(parts.cells, dtype=torch.int64, device=device).view(h, LANES, 4)
    rows = torch.arange(h, device=pos.device).view(h, 1, 1)
    if not bool((pos // STRIP == rows).all()):
        raise UnsupportedNode("cell order must keep every tile row in its own ring row "
                              "(row-preserving permutation of each row's 128 cells)")
    col = pos - rows * STRIP
    if not bool((col[..., 0] % 4 == 0).all()) or not bool((col - col[..., :1] ==
                                                            torch.arange(4, device=pos.device)).all()):
        raise UnsupportedNode("cell order must move each lane's 4-column group as one aligned, "
                              "contiguous 16-byte group")
    slots = torch.sort(col[..., 0] // 4, dim=1).values
    if not torch.equal(slots, torch.arange(LANES, device=pos.device).expand(h, LANES)):
        raise UnsupportedNode("cell order is not a permutation of each row's lane groups")
    host = pos.view(-1).cpu().tolist()
    for x in _host_points(h * STRIP):
        r, c = divmod(x, STRIP)
        if parts.cells.apply((r, c)) != host[x]:
            raise UnsupportedNode(f"cell order: concrete apply({r}, {c}) != generated {host[x]}")


# ---------------------------------------------------------------------------
# program
# ---------------------------------------------------------------------------

def needs_program(defines: dict) -> bool:
    """Whether a layout's program differs from the library's built-in strip
    instance (tiles, a generated tile order or a generated cell order); the
    tuning defines (NW_SKEW, NW_GRP) do not count."""
    return any(defines.get(k) for k in ("NW_TILED", "NW_GEN_TILES", "NW_GEN_SLOTS"))


def program_source(parts: NwParts) -> Tuple[str, runtime.ProgramInfo, dict]:
    """NVRTC source of the wavefront specialised to the layout's maps."""
    from .kernels import _text
    nt = parts.nr * parts.nc
    body = codegen.constant("NR", parts.nr) + codegen.constant("NC", parts.nc)
    body += codegen.constant("H", parts.h)
    gen_tiles = gen_slots = 0
    if nt > 1:
        f, inv = lower.inv_map_expr(parts.tiles)
        if lower.simplify(inv - f) != IntConst(0):
            gen_tiles = 1
            body += codegen.generate("tile_of", [f], {"x": inv}, bounds={"x": (0, nt - 1)}).source
    r = Var("r", VarRange(0, parts.h))
    g = Var("g", VarRange(0, LANES))
    s = _slot_expr(parts, r, g)
    if lower.simplify(s - g) != IntConst(0):
        gen_slots = 1
        body += codegen.generate("slot", [r, g], {"s": s}, bounds={"s": (0, LANES - 1)}).source
    tiled = int(parts.nr > 1)
    # lanes one row apart (skew 1) unless tiles are tall, and the boundary
    # readiness check every 4 steps in tiled programs (every 2 in strips).
    # Measured at n = 16384 (scripts/ab_nw.py): 4096-row tiles skew 2 / check
    # every 4: 1212 us (skew 2 / 2: 1320, skew 1 / 4: 1279, skew 1 / 2: 1394);
    # 128-row tiles skew 1 / 4: 1586 (skew 1 / 2: 1646, skew 2 / 4: 1768);
    # strips skew 1 / 2: 882 (skew 1 / 4: 897)
    skew = 2 if tiled and parts.h >= 2048 else 1
    defines = {"NW_TILED": tiled, "NW_GEN_TILES": gen_tiles, "NW_GEN_SLOTS": gen_slots, "NW_SKEW": skew,
               "NW_GRP": 4 if tiled else 2}
    head = "".join(f"#ifndef {k}\n#define {k} {v}\n#endif\n" for k, v in defines.items())
    src = (head + _text("lego_index.cuh").replace("#pragma once", "") + "\nnamespace gen {\n" + body + "}\n"
           + _text("nw_kernels.cuh").replace("#pragma once", ""))
    info = runtime.ProgramInfo(kind=KIND_NW, elem_bytes=4, n=parts.n, units=parts.h,
                               unit_threads=parts.nr, block=128, smem_bytes=SMEM_BYTES, reserved=tiled)
    return src, info, defines


def nw_program(layout, n: int, device=None):
    """Prove and compile (cached per layout, n and device by kernels'
    program cache; equal generated sources share one loaded module).  The
    returned program carries ``parts`` and ``defines``."""
    import torch

    from . import kernels as K
    dev = K._device(device)

    def build():
        parts = nw_parts(layout, n)
        check_tile_order(parts, device=dev)
        check_cell_order(parts, device=dev)
        src, info, defines = program_source(parts)
        return src, info, {"parts": parts, "defines": defines}

    with torch.cuda.device(dev):
        return K._program(("nw", K._layout_key(layout), n), build, dev.index)


def describe(layout) -> str:
    """Short text of an NW layout (for bench lines and errors)."""
    parts = []
    for stage in layout.orders:
        parts.append("OrderBy(" + ", ".join(_perm_text(p) for p in stage.perms) + ")")
    return f"GroupBy([{', '.join(map(str, layout.dims))}])." + ".".join(parts)


def _perm_text(p) -> str:
    if isinstance(p, RegP):
        return f"RegP({list(p.shape)}, {list(p.sigma)})"
    return f"GenP({list(p.shape)}, {p.name or 'user'})"

