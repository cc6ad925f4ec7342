"""User-defined bijections (GenP + PermFn, reference layout.py:152-200) for
the parity tests of arbitrary user permutations at scale.

Each factory takes the layout module ``L`` -- the reference package
(``lego``, for tests/golden/make_user_golden.py) or the backend's mirror
(``paper_2505_08091_b200``) -- and builds the same layout from the same
concrete callables and symbolic builders, the way a user would write them:

* ``xor_swizzle``  -- (i, j) of 1024 x 1024 -> i*1024 + (j XOR i)
* ``bit_reverse``  -- x of 2^20 -> x with its 20 bits reversed
* ``morton``       -- (i, j) of 1024 x 1024 -> bits of i and j interleaved
* ``skew``         -- (a, b) of 512 x 2048 -> anti-diagonal order of a rectangle
* ``even_map``     -- x of 2^20 -> 2x (injective mode: apply only)
* ``tiled_xor``    -- 2048 x 512 in 64 x 64 tiles (tile-major, tiles transposed),
                      each tile XOR-swizzled: a chain with an in-tile user GenP

All but ``even_map`` are bijections of 2^20 points, far above the
4096-point bound up to which the reference's ``validate`` enumerates a GenP.
"""

from __future__ import annotations

import math


def _bits(x, k):
    return [(x // (1 << b)) % 2 for b in range(k)]


def _xor(a, b, k):
    """a XOR b for 0 <= a, b < 2^k using only +, //, % (ints and Exprs)."""
    return sum(((ba + bb) % 2) * (1 << i) for i, (ba, bb) in enumerate(zip(_bits(a, k), _bits(b, k))))


def xor_swizzle(L, n=1024):
    k = n.bit_length() - 1

    def fwd(idx):
        i, j = idx
        return i * n + (j ^ (i % n))

    def fwd_sym(idx):
        i, j = idx
        return i * n + _xor(j, i % n, k)

    def inv(f):
        return f // n, (f % n) ^ ((f // n) % n)

    def inv_sym(f):
        return f // n, _xor(f % n, (f // n) % n, k)

    g = L.GenP((n, n), L.PermFn(fwd, fwd_sym), L.PermFn(inv, inv_sym))
    return L.GroupBy([n, n], orders=(L.OrderBy(g),))


def bit_reverse(L, k=20):
    n = 1 << k

    def rev(x):
        return sum(((x >> b) & 1) << (k - 1 - b) for b in range(k))

    def rev_sym(x):
        return sum(((x // (1 << b)) % 2) * (1 << (k - 1 - b)) for b in range(k))

    g = L.GenP((n,), L.PermFn(lambda idx: rev(idx[0]), lambda idx: rev_sym(idx[0])),
               L.PermFn(lambda f: (rev(f),), lambda f: (rev_sym(f),)))
    return L.GroupBy([n], orders=(L.OrderBy(g),))


def morton(L, n=1024):
    k = n.bit_length() - 1

    def fwd(idx):
        i, j = idx
        return sum((((i >> b) & 1) << (2 * b + 1)) | (((j >> b) & 1) << (2 * b)) for b in range(k))

    def fwd_sym(idx):
        i, j = idx
        return sum(((i // (1 << b)) % 2) * (1 << (2 * b + 1)) + ((j // (1 << b)) % 2) * (1 << (2 * b))
                   for b in range(k))

    def inv(f):
        return (sum(((f >> (2 * b + 1)) & 1) << b for b in range(k)),
                sum(((f >> (2 * b)) & 1) << b for b in range(k)))

    def inv_sym(f):
        return (sum(((f // (1 << (2 * b + 1))) % 2) * (1 << b) for b in range(k)),
                sum(((f // (1 << (2 * b))) % 2) * (1 << b) for b in range(k)))

    g = L.GenP((n, n), L.PermFn(fwd, fwd_sym), L.PermFn(inv, inv_sym))
    return L.GroupBy([n, n], orders=(L.OrderBy(g),))


def _tri(d):
    return (d * (d + 1)) // 2


def skew(L, R=512, C=2048):
    m, M = min(R, C), max(R, C)
    total = R * C
    head = _tri(m)
    body = head + (M - m) * m

    def fwd(idx):
        a, b = idx
        d = a + b
        if d < m:
            st = _tri(d)
        elif d < M:
            st = head + (d - m) * m
        else:
            st = total - _tri(R + C - 1 - d)
        return st + a - max(0, d - (C - 1))

    def fwd_sym(idx):
        a, b = idx
        d = a + b
        st = L.Select(L.lt(d, m), _tri(d), L.Select(L.lt(d, M), head + (d - m) * m,
                                                    total - _tri((R + C - 1) - d)))
        return st + a - L.Select(L.lt(d, C), 0, d - (C - 1))

    def inv(f):
        if f < head:
            d = (math.isqrt(8 * f + 1) - 1) // 2
            a = f - _tri(d)
            return a, d - a
        if f < body:
            d = m + (f - head) // m
            a = max(0, d - (C - 1)) + (f - head) % m
            return a, d - a
        g = total - 1 - f
        d = (math.isqrt(8 * g + 1) - 1) // 2
        a2 = g - _tri(d)
        return R - 1 - a2, C - 1 - (d - a2)

    def inv_sym(f):
        in_head, in_body = L.lt(f, head), L.lt(f, body)
        x = L.Select(in_head, f, (total - 1) - f)
        d1 = (L.isqrt(8 * x + 1) - 1) // 2
        i1 = x - _tri(d1)
        db = m + (f - head) // m
        ab = L.Select(L.lt(db, C), 0, db - (C - 1)) + (f - head) % m
        a = L.Select(in_head, i1, L.Select(in_body, ab, (R - 1) - i1))
        b = L.Select(in_head, d1 - i1, L.Select(in_body, db - ab, (C - 1) - (d1 - i1)))
        return a, b

    g = L.GenP((R, C), L.PermFn(fwd, fwd_sym), L.PermFn(inv, inv_sym))
    return L.GroupBy([R, C], orders=(L.OrderBy(g),))


def even_map(L, n=1 << 20):
    g = L.GenP((n,), L.PermFn(lambda idx: 2 * idx[0], lambda idx: 2 * idx[0]), None)
    return L.GroupBy([n], orders=(L.OrderBy(g),), injective=True)


def tiled_xor(L, rows=2048, cols=512, t=64):
    k = t.bit_length() - 1

    def fwd(idx):
        r, c = idx
        return r * t + (c ^ (r % t))

    def fwd_sym(idx):
        r, c = idx
        return r * t + _xor(c, r % t, k)

    def inv(f):
        return f // t, (f % t) ^ ((f // t) % t)

    def inv_sym(f):
        return f // t, _xor(f % t, (f // t) % t, k)

    g = L.GenP((t, t), L.PermFn(fwd, fwd_sym), L.PermFn(inv, inv_sym))
    tr, tc = rows // t, cols // t
    return L.GroupBy([rows, cols], orders=(L.OrderBy(L.RegP([tr, t, tc, t], [1, 3, 2, 4])),
                                           L.OrderBy(L.RegP([tr, tc], [2, 1]), g)))


FACTORIES = {"xor_swizzle": xor_swizzle, "bit_reverse": bit_reverse, "morton": morton, "skew": skew,
             "even_map": even_map, "tiled_xor": tiled_xor}
