"""The GEMM's data, thread and shared-memory layouts written as LEGO layouts.

* ``raster_layout(mb, nb, g)`` -- the CTA tile raster walked by
  ``csrc/gemm_tcgen05.cu`` when g divides mb (``tile_coords`` evaluates its
  inverse); ``grouped_raster_perm(mb, nb, g)`` -- the same order for any mb,
  a user-defined GenP over the (m-block, n-block) grid whose last group
  holds the mb % g remaining m-blocks (tests/test_gemm_raster.py compares
  both with the device's tile order).
* ``sw128_perm()`` -- the 128-byte shared-memory swizzle that TMA
  (``CU_TENSOR_MAP_SWIZZLE_128B``) writes and the UMMA descriptors
  (layout type 2) read: inside a 1024-byte atom of 8 rows x 8 16-byte chunks,
  chunk ``c`` of row ``r`` sits at chunk ``c XOR r``.  A user-defined LEGO
  bijection (``GenP``) whose symbolic builder spells XOR with ``//`` and ``%``
  on the three chunk bits, so the CUDA code generator can emit it.
* ``kmajor_smem_layout(rows, k)`` -- a K-major bf16 operand tile
  (``rows`` x ``k``, k = 64 per 128-byte row) in that swizzle:
  ``GroupBy([rows/8, 8, 8, 8]).OrderBy(Row(rows/8), GenP([8,8], sw128), Row(8))``
  over (row_hi, row_lo, chunk, element).
"""

from __future__ import annotations

from .dsl import parse_layout
from .expr import Select, lt
from .layout import GenP, GroupBy, OrderBy, PermFn, RegP


def _xor3(a, b):
    """a XOR b for 0 <= a, b < 8, with only +, //, % (works on ints and Exprs)."""
    return sum((((a // (1 << k)) % 2 + (b // (1 << k)) % 2) % 2) * (1 << k) for k in range(3))


def sw128_perm() -> GenP:
    """(row r, chunk c) of an 8 x 8 atom -> r*8 + (c XOR r)."""
    def fwd(idx):
        r, c = idx
        return r * 8 + (c ^ r)

    def fwd_sym(idx):
        r, c = idx
        return r * 8 + _xor3(c, r)

    def inv(flat):
        r, x = divmod(flat, 8)
        return r, x ^ r

    def inv_sym(flat):
        r = flat // 8
        return r, _xor3(flat % 8, r)

    return GenP((8, 8), PermFn(fwd, fwd_sym), PermFn(inv, inv_sym), name="sw128")


def kmajor_smem_layout(rows: int, k: int = 64) -> GroupBy:
    """Element offsets of a K-major bf16 tile (rows x k, 128-byte rows) in the
    SWIZZLE_128B layout; k must be 64 (one swizzle row of bf16)."""
    if rows % 8 or k != 64:
        raise ValueError("rows % 8 == 0 and k == 64 (bf16 128-byte swizzle rows)")
    return GroupBy([rows // 8, 8, 8, 8], orders=(OrderBy(RegP([rows // 8], [1]), sw128_perm(),
                                                         RegP([8], [1])),))


def raster_layout(mb: int, nb: int, g: int) -> GroupBy:
    """Tile raster: tile t -> (group, n-block, m within group), m fastest."""
    return parse_layout(f"GroupBy([{mb // g},{nb},{g}]).OrderBy(Row({mb // g},{nb},{g}))")


def grouped_raster_perm(mb: int, nb: int, g: int) -> GenP:
    """Tile (m, n) -> rank t of the grouped raster: groups of g m-blocks, each
    walked n-major with m fastest; a last group of mb % g m-blocks."""
    full = (mb // g) * g
    tail = mb - full

    def fwd(idx):
        m, n = idx
        if m < full:
            return ((m // g) * nb + n) * g + m % g
        return full * nb + n * tail + (m - full)

    def fwd_sym(idx):
        m, n = idx
        t_tail = (m - full) + n * tail + full * nb
        return Select(lt(m, full), ((m // g) * nb + n) * g + m % g, t_tail) if tail else \
            ((m // g) * nb + n) * g + m % g

    def inv(t):
        if t < full * nb:
            grp, rem = divmod(t, g * nb)
            return grp * g + rem % g, rem // g
        rem = t - full * nb
        return full + rem % tail, rem // tail

    def inv_sym(t):
        rem = t % (g * nb)
        m_full, n_full = (t // (g * nb)) * g + rem % g, rem // g
        if not tail:
            return m_full, n_full
        r2 = t - full * nb
        head = lt(t, full * nb)
        return Select(head, m_full, full + r2 % tail), Select(head, n_full, r2 // tail)

    return GenP((mb, nb), PermFn(fwd, fwd_sym), PermFn(inv, inv_sym), name=None)


def operand_strides(layout):
    """(s_i, s_j) with ``layout.apply((i, j)) == i*s_i + j*s_j`` for every
    logical (i, j) of a 2-D data layout -- the affine form a single-RegP
    ``OrderBy`` always has (paper Table I; reference test_acceptance.py:167-208).
    The tcgen05 GEMM feeds an operand to TMA from exactly these strides, so
    this is how a LEGO ``Data`` layout (reference matmul workflow,
    test_acceptance.py:211-234) drives the operand addressing.  Raises
    ``UnsupportedNode`` for non-affine layouts."""
    from .errors import UnsupportedNode
    from .expr import IntConst
    from .layout import apply_symbolic, index_vars
    from .simplify import simplify
    if len(layout.dims) != 2:
        raise UnsupportedNode("a GEMM operand layout is 2-D")
    i, j = index_vars(["i", "j"], layout.dims)
    e = simplify(apply_symbolic(layout, (i, j)))
    c = layout.apply((0, 0))
    s_i = layout.apply((1, 0)) - c if layout.dims[0] > 1 else 0
    s_j = layout.apply((0, 1)) - c if layout.dims[1] > 1 else 0
    if c != 0 or simplify(e - (i * s_i + j * s_j)) != IntConst(0):
        raise UnsupportedNode(f"operand layout is not affine (i*{s_i} + j*{s_j}): {layout!r}")
    return s_i, s_j


def operand_major(layout, what: str) -> str:
    """'row' when the second logical index has stride 1 (row-major storage),
    'col' when the first has (column-major), for an affine 2-D layout."""
    from .errors import UnsupportedNode
    rows, cols = layout.dims
    s_i, s_j = operand_strides(layout)
    if (s_i, s_j) == (cols, 1):
        return "row"
    if (s_i, s_j) == (1, rows):
        return "col"
    raise UnsupportedNode(f"{what}: strides ({s_i}, {s_j}) are neither row- nor column-major")
