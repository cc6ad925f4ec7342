"""Seeded generator of random LEGO layout DSL strings (tiled GroupBy + 1-2
OrderBy stages of RegP / Row / Col / GenP(antidiag | rev2d) perms), used by the
CPU frontend-vs-oracle test and the GPU parity test.  Sizes stay <= 8192."""

import random


def _factor(n, rng):
    ds = [d for d in range(2, n) if n % d == 0]
    if not ds:
        return None
    a = rng.choice(ds)
    return a, n // a


def _perm(dims, rng):
    """One perm over exactly `dims` (a list of extents)."""
    k = len(dims)
    choice = rng.random()
    if k == 2 and dims[0] == dims[1] and choice < 0.3:
        return f"GenP([{dims[0]},{dims[1]}], {rng.choice(['antidiag', 'rev2d'])})"
    if choice < 0.5:
        sigma = list(range(1, k + 1))
        rng.shuffle(sigma)
        return f"RegP([{','.join(map(str, dims))}],[{','.join(map(str, sigma))}])"
    if choice < 0.75:
        return f"Row({','.join(map(str, dims))})"
    return f"Col({','.join(map(str, dims[::-1]))})"      # Col takes memory-order extents


def random_layout(rng):
    d = rng.choice([1, 2, 2, 2, 3])
    while True:
        ext = [rng.choice([2, 3, 4, 5, 6, 8, 9, 12, 16, 24, 32]) for _ in range(d)]
        size = 1
        for e in ext:
            size *= e
        if 4 <= size <= 8192:
            break
    # optional tiling: split each extent into outer x inner
    tiles = [ext]
    if rng.random() < 0.6:
        outer, inner = [], []
        for e in ext:
            f = _factor(e, rng)
            if f is None:
                outer.append(1)
                inner.append(e)
            else:
                outer.append(f[0])
                inner.append(f[1])
        if all(o > 1 for o in outer):
            tiles = [outer, inner]
    dims = [n for t in tiles for n in t]
    text = "GroupBy(" + ", ".join("[" + ",".join(map(str, t)) + "]" for t in tiles) + ")"
    for _ in range(rng.choice([1, 1, 2])):
        if len(dims) >= 2 and rng.random() < 0.5:
            cut = rng.randrange(1, len(dims))
            text += f".OrderBy({_perm(dims[:cut], rng)}, {_perm(dims[cut:], rng)})"
        else:
            text += f".OrderBy({_perm(dims, rng)})"
    return text


def corpus(count=60, seed=20261017):
    rng = random.Random(seed)
    return [random_layout(rng) for _ in range(count)]


def random_expand(rng):
    """ExpandBy(physical, expanded, inner): partial tiles of a random tiled layout."""
    while True:
        inner = random_layout(rng)
        if not inner.startswith("GroupBy("):
            continue
        import re
        tiles = [list(map(int, t.split(","))) for t in re.findall(r"\[([0-9,]+)\]", inner.split(".")[0])]
        k = len(tiles[0])
        expanded = [1] * k
        for t in tiles:
            expanded = [a * b for a, b in zip(expanded, t)]
        physical = [max(1, e - rng.randrange(0, max(1, e // 3) + 1)) for e in expanded]
        return (f"ExpandBy([{','.join(map(str, physical))}],[{','.join(map(str, expanded))}],{inner})")


def expand_corpus(count=24, seed=20261018):
    rng = random.Random(seed)
    return [random_expand(rng) for _ in range(count)]


def _tile_perm(a, b, rng):
    """A perm over an (a, b) tile: antidiag / rev2d when square, else a RegP/Row/Col."""
    if a == b and rng.random() < 0.5:
        return f"GenP([{a},{b}], {rng.choice(['antidiag', 'rev2d'])})"
    return rng.choice([f"RegP([{a},{b}],[2,1])", f"Row({a},{b})", f"Col({b},{a})"])


def tiled_chain(rng):
    """SURVEY f1-style two-stage chain at up to 2^20 points: tile a (M x N)
    matrix by (a x b), then reorder the tile grid and the in-tile elements."""
    while True:
        a = rng.choice([8, 16, 32, 64, 24, 48])
        b = rng.choice([a, a, 16, 32, 64])
        gm = rng.choice([2, 4, 8, 16, 3, 6])
        gn = rng.choice([2, 4, 8, 16, 5])
        if a * b * gm * gn <= 1 << 20:
            break
    M, N = a * gm, b * gn
    text = (f"GroupBy([{M},{N}]).OrderBy(RegP([{gm},{a},{gn},{b}],[1,3,2,4]))"
            f".OrderBy({_tile_perm(gm, gn, rng)}, {_tile_perm(a, b, rng)})")
    return text


def chain_corpus(count=16, seed=20261019):
    rng = random.Random(seed)
    return [tiled_chain(rng) for _ in range(count)]
