"""User-defined LEGO permutations (GenP + PermFn, reference layout.py:152-200)
used as NW tile orders and shared-memory cell orders in the tests and the
bench.  None of these is a built-in: each is a concrete callable plus a
symbolic builder written the way a user of the reference package would.

* :func:`skew_order` -- anti-diagonal order of a rectangular R x C grid
  (diagonal d = a + b, then a), the rectangular generalisation of the
  built-in square ``antidiag`` (which needs R == C);
* :func:`morton_order` -- Z-order (bit interleave) of a 2^k x 2^k grid;
* :func:`rotate_cells` -- lane group g of row r stored at slot (g + r) % 32;
* :func:`xor_cells` -- lane group g of row r stored at slot g XOR (r % 32).
"""

from __future__ import annotations

import math

from paper_2505_08091_b200 import GenP, PermFn, Select, isqrt, lt


def _tri(d):
    return (d * (d + 1)) // 2


def skew_order(rows: int, cols: int) -> GenP:
    """Position of tile (a, b): all tiles of earlier anti-diagonals, then a."""
    R, C = rows, cols
    m, M = min(R, C), max(R, C)
    total = R * C
    head = _tri(m)                       # positions of the growing triangle
    body = head + (M - m) * m            # + the constant-width band

    def start(d):                        # first position of diagonal d
        if d < m:
            return _tri(d)
        if d < M:
            return head + (d - m) * m
        u = R + C - 1 - d
        return total - _tri(u)

    def fwd(idx):
        a, b = idx
        d = a + b
        return start(d) + a - max(0, d - (C - 1))

    def fwd_sym(idx):
        a, b = idx
        d = a + b
        u = (R + C - 1) - d
        st = Select(lt(d, m), _tri(d), Select(lt(d, M), head + (d - m) * m, total - _tri(u)))
        amin = Select(lt(d, C), 0, d - (C - 1))
        return st + a - amin

    def tri_root(x):                     # largest d with d(d+1)/2 <= x
        return (math.isqrt(8 * x + 1) - 1) // 2

    def inv(f):
        if f < head:
            d = tri_root(f)
            a = f - _tri(d)
            return a, d - a
        if f < body:
            d = m + (f - head) // m
            i = (f - head) % m
            a = max(0, d - (C - 1)) + i
            return a, d - a
        g = total - 1 - f                # point reflection: same order on the reversed grid
        d = tri_root(g)
        a2 = g - _tri(d)
        b2 = d - a2
        return R - 1 - a2, C - 1 - b2

    def inv_sym(f):
        in_head = lt(f, head)
        in_body = lt(f, body)
        g = (total - 1) - f
        x = Select(in_head, f, g)
        d1 = (isqrt(8 * x + 1) - 1) // 2
        i1 = x - _tri(d1)
        j1 = d1 - i1
        db = m + (f - head) // m
        ib = (f - head) % m
        ab = Select(lt(db, C), 0, db - (C - 1)) + ib
        a = Select(in_head, i1, Select(in_body, ab, (R - 1) - i1))
        b = Select(in_head, j1, Select(in_body, db - ab, (C - 1) - j1))
        return a, b

    return GenP((R, C), PermFn(fwd, fwd_sym), PermFn(inv, inv_sym), name=None)


def morton_order(side: int) -> GenP:
    """Z-order of a side x side grid (side a power of two): bits of a and b
    interleaved, a's bit above b's."""
    k = side.bit_length() - 1
    if side != 1 << k:
        raise ValueError("morton_order needs a power-of-two side")

    def fwd(idx):
        a, b = idx
        return sum((((a >> j) & 1) << (2 * j + 1)) | (((b >> j) & 1) << (2 * j)) for j in range(k))

    def fwd_sym(idx):
        a, b = idx
        out = 0
        for j in range(k):
            out = out + ((a // (1 << j)) % 2) * (1 << (2 * j + 1)) + ((b // (1 << j)) % 2) * (1 << (2 * j))
        return out

    def inv(f):
        a = sum(((f >> (2 * j + 1)) & 1) << j for j in range(k))
        b = sum(((f >> (2 * j)) & 1) << j for j in range(k))
        return a, b

    def inv_sym(f):
        a = 0
        b = 0
        for j in range(k):
            a = a + ((f // (1 << (2 * j + 1))) % 2) * (1 << j)
            b = b + ((f // (1 << (2 * j))) % 2) * (1 << j)
        return a, b

    return GenP((side, side), PermFn(fwd, fwd_sym), PermFn(inv, inv_sym), name=None)


def rotate_cells(h: int) -> GenP:
    """Cells of an h x 128 tile: row r, column 4g + k -> r*128 + 4*((g + r) % 32) + k."""
    def fwd(idx):
        r, c = idx
        return r * 128 + 4 * ((c // 4 + r) % 32) + c % 4

    def inv(f):
        r, x = divmod(f, 128)
        return r, 4 * ((x // 4 - r) % 32) + x % 4

    def inv_sym(f):
        r = f // 128
        x = f % 128
        return r, 4 * ((x // 4 - r) % 32) + x % 4

    return GenP((h, 128), PermFn(fwd, fwd), PermFn(inv, inv_sym), name=None)


def _xor5(a, b):
    """a XOR b for 0 <= a, b < 32 with only +, //, % (ints and Exprs)."""
    return sum((((a // (1 << k)) % 2 + (b // (1 << k)) % 2) % 2) * (1 << k) for k in range(5))


def xor_cells(h: int) -> GenP:
    """Cells of an h x 128 tile: row r, column 4g + k -> r*128 + 4*(g XOR (r % 32)) + k."""
    def fwd(idx):
        r, c = idx
        return r * 128 + 4 * ((c // 4) ^ (r % 32)) + c % 4

    def fwd_sym(idx):
        r, c = idx
        return r * 128 + 4 * _xor5(c // 4, r % 32) + c % 4

    def inv(f):
        r, x = divmod(f, 128)
        return r, 4 * ((x // 4) ^ (r % 32)) + x % 4

    def inv_sym(f):
        r = f // 128
        x = f % 128
        return r, 4 * _xor5(x // 4, r % 32) + x % 4

    return GenP((h, 128), PermFn(fwd, fwd_sym), PermFn(inv, inv_sym), name=None)


def nw_test_layouts(n: int):
    """(name, layout) pairs exercised by tests/test_nw_layouts.py at size n:
    the default strip layout plus tiled layouts with built-in and user
    tile orders and user cell orders (precompiled by __graft_entry__.build)."""
    from paper_2505_08091_b200.nw import nw_layout
    out = [("strips", nw_layout(n))]
    if n <= 128:
        out.append(("strips+rotate", nw_layout(n, cell_order=rotate_cells(max(n, 1)))))
        out.append(("strips+xor", nw_layout(n, tile_rows=128, cell_order=xor_cells(128))))
    elif n <= 2048:                                  # user cell order where the 256-row ring wraps
        out.append(("strips+rotate", nw_layout(n, cell_order=rotate_cells(n))))
    if n > 32:
        h = 32 if n <= 128 else 128
        nr, nc = -(-n // h), -(-n // 128)
        out.append((f"tiles{h}+skew+rotate", nw_layout(n, tile_rows=h, tile_order=skew_order(nr, nc),
                                                        cell_order=rotate_cells(h))))
        if nr == nc:
            out.append((f"tiles{h}+antidiag", nw_layout(n, tile_rows=h, tile_order="antidiag")))
            if nr & (nr - 1) == 0:
                out.append((f"tiles{h}+morton", nw_layout(n, tile_rows=h, tile_order=morton_order(nr))))
    if n >= 1024:
        h = n // 8
        out.append((f"tiles{h}+col", nw_layout(n, tile_rows=h, tile_order="col")))
    if n >= 16384:                                   # the bench's user-ordered layout
        out.append(("tiles4096+skew", nw_layout(n, tile_rows=4096, tile_order=skew_order(n // 4096, n // 128))))
    return out
