"""Build product layouts from golden specs (test helper, independent of the
oracle's own parser)."""

import paper_2505_08091_b200 as L


def _perm(p):
    shape = tuple(p["shape"])
    if p["kind"] == "regp":
        return L.RegP(shape, tuple(p["sigma"]))
    if p["kind"] == "identity":
        return L.identity_perm(shape)
    if p["kind"] == "rev":
        return L.reverse_perm(shape)
    if p["kind"] == "antidiag":
        return L.antidiag_perm(shape[0])
    raise ValueError(p)


def layout_from_spec(spec):
    if spec["kind"] == "expand":
        return L.ExpandBy(tuple(spec["physical"]), tuple(spec["expanded"]),
                          layout_from_spec(spec["inner"]))
    orders = tuple(L.OrderBy(*[_perm(p) for p in st]) for st in spec["stages"])
    return L.GroupBy(*[tuple(t) for t in spec["tiles"]], orders=orders)


def unflat(shape, f):
    out = []
    for n in reversed(shape[1:]):
        out.append(f % n)
        f //= n
    out.append(f)
    return tuple(out[::-1])


def flat(shape, idx):
    acc = 0
    for c, n in zip(idx, shape):
        acc = acc * n + c
    return acc
