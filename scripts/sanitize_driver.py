"""One small launch of every kernel family, for compute-sanitizer runs
(scripts/sanitize.sh): remap kinds 1-5 (+ routed, + TMA-bulk staged), index
maps, bijectivity histogram, softmax, NW, GEMM.  Checks results against the
oracle so a sanitizer run is also a parity run."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2505_08091_b200 as L  # noqa: E402
from paper_2505_08091_b200 import kernels as K, shard, staging  # noqa: E402
from oracle import oracle as O  # noqa: E402


def check_remap(text, elem_dt, np_dt, src_side=False):
    g = L.parse_layout(text)
    spec = O.parse(text)
    n = O.logical_size(spec) if not src_side else O.size(spec)
    host = (np.arange(n, dtype=np.int64) * 7919 % 30011).astype(np_dt)
    src_l, dst_l = (g, None) if src_side else (None, g)
    got = K.remap(torch.from_numpy(host).cuda(), src_l, dst_l).cpu().numpy()
    want = O.remap(host, spec if src_side else None, None if src_side else spec,
                   dst_size=O.logical_size(spec) if src_side else O.size(spec))
    assert np.array_equal(got, want), text
    return repr(K.remap_plan(src_l, dst_l, np.dtype(np_dt).itemsize))


plans = []
for text, src_side in (
        ("GroupBy([256,256]).OrderBy(Col(256,256))", False),                         # transpose
        ("GroupBy([128,128]).OrderBy(RegP([4,32,4,32],[1,3,2,4]))", False),          # gather
        ("GroupBy([256,256]).OrderBy(GenP([256,256], antidiag))", False),            # band scatter
        ("GroupBy([256,256]).OrderBy(GenP([256,256], antidiag))", True),             # band gather
        ("GroupBy([256,256]).OrderBy(RegP([4,64,4,64],[1,3,2,4])).OrderBy(RegP([4,4],[2,1]), "
         "GenP([64,64], antidiag))", False),                                         # staged
        ("GroupBy([256,256]).OrderBy(RegP([4,64,4,64],[1,3,2,4])).OrderBy(RegP([4,4],[2,1]), "
         "GenP([64,64], antidiag))", True),                                          # staged mirrored
        ("GroupBy([30,30]).OrderBy(Col(30,30))", False),                             # ragged scalar
        ("ExpandBy([30,28],[32,32],GroupBy([32,32]).OrderBy(RegP([2,16,2,16],[1,3,2,4])))", True)):
    for dt in (np.int16, np.int32):
        plans.append(check_remap(text, None, dt, src_side))
# register interleaves (AoS <-> AoSoA, 1- and 2-byte elements, both directions)
for text in ("GroupBy([512,32,4]).OrderBy(RegP([512,32,4],[1,3,2]))",
             "GroupBy([1024,32,2]).OrderBy(RegP([1024,32,2],[1,3,2]))"):
    for dt in (np.int8, np.int16):
        for side in (False, True):
            plans.append(check_remap(text, None, dt, side))
staging.BOX_BULK = 1
plans.append(check_remap("GroupBy([256,256]).OrderBy(RegP([4,64,4,64],[1,3,2,4])).OrderBy(RegP([4,4],[2,1]), "
                         "GenP([64,64], antidiag))", None, np.int32))
staging.BOX_BULK = 0
# injective scatter
even = L.GenP((1024,), L.PermFn(lambda i: i[0] * 2, lambda i: i[0] * 2), None, name="even")
gi = L.GroupBy([1024], orders=(L.OrderBy(even),), injective=True)
out = K.remap(torch.arange(1024, dtype=torch.int32, device="cuda"), None, gi).cpu().numpy()
assert np.array_equal(out[0::2], np.arange(1024)) and not out[1::2].any()
# routed transpose (emulated peers)
world, R, C = 2, 64, 128
full = torch.arange(world * R * world * C, device="cuda", dtype=torch.int32).reshape(world * R, world * C)
shards = [torch.zeros(C, world * R, dtype=torch.int32, device="cuda") for _ in range(world)]
peers = torch.tensor([t.data_ptr() for t in shards], dtype=torch.int64, device="cuda")
for r in range(world):
    lay, route = shard.fused_transpose_route(R, C, world, r)
    K.remap_routed(full[r * R:(r + 1) * R].reshape(-1), None, lay, peers, route)
assert all(torch.equal(shards[q], full.t()[q * C:(q + 1) * C]) for q in range(world))
# index maps + bijectivity
ga = L.parse_layout("GroupBy([96,96]).OrderBy(GenP([96,96], antidiag))")
assert np.array_equal(K.apply_map(ga).cpu().numpy(), O.apply_range(O.parse("GroupBy([96,96]).OrderBy(GenP([96,96], antidiag))")))
assert np.array_equal(K.inv_map(ga).cpu().numpy(), O.inv_range(O.parse("GroupBy([96,96]).OrderBy(GenP([96,96], antidiag))")))
assert K.check_bijective(ga)
# softmax (vector and ragged)
for rows, cols in ((16, 1024), (5, 33)):
    x = torch.randn(rows, cols, device="cuda")
    y = K.softmax(x).cpu().numpy()
    want = O.softmax_rows_f64(x.cpu().numpy())
    assert np.abs(y - want).max() / want.max() < 1e-5
# NW (vector and ragged widths)
for n in (64, 100):
    sim = np.random.default_rng(n).integers(-10, 11, size=(n, n), dtype=np.int32)
    assert np.array_equal(K.nw_score(torch.from_numpy(sim).cuda(), 10).cpu().numpy(), O.nw(sim, 10))
# GEMM (pair kernel, ragged)
for M, N_, Kd in ((256, 256, 128), (200, 136, 72)):
    a = torch.randn(M, Kd, device="cuda").to(torch.bfloat16)
    b = torch.randn(N_, Kd, device="cuda").to(torch.bfloat16)
    c = K.gemm(a, b).float()
    ref = a.float() @ b.float().t()
    assert ((c - ref).abs().max() / ref.abs().max()).item() < 1e-2
# round 2: fill-mode scatters (fused affine windows, fill pass + scatter), the
# device injectivity gate, the run-walking antidiag inverse, the generated
# softmax program, NW layout programs (tiled, user orders), a user template
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
for f in (lambda x: 2 * x, lambda x: x * x):
    gf = L.GroupBy([1 << 12], orders=(L.OrderBy(L.GenP((1 << 12,), L.PermFn(lambda i, f=f: f(i[0]),
                                                                               lambda i, f=f: f(i[0])), None)),),
                   injective=True)
    x = torch.arange(1 << 12, dtype=torch.int32, device="cuda")
    got = K.remap(x, None, gf, fill=-1).cpu().numpy()
    want = np.full(got.size, -1, np.int32)
    want[[f(v) for v in range(1 << 12)]] = np.arange(1 << 12)
    assert np.array_equal(got, want)
big = L.GroupBy([1 << 13], orders=(L.OrderBy(L.GenP((1 << 13,), L.PermFn(lambda i: 3 * i[0], lambda i: 3 * i[0]),
                                                  None)),), injective=True)
assert K.check_injective(big)
K.remap(torch.arange(1 << 13, dtype=torch.int16, device="cuda"), None, big)          # gated scatter
g4 = L.parse_layout("GroupBy([512,512]).OrderBy(GenP([512,512], antidiag))")
assert np.array_equal(K.inv_map(g4).cpu().numpy(), O.inv_range(O.parse("GroupBy([512,512]).OrderBy(GenP([512,512], antidiag))")))
x = torch.randn(6, 2048, device="cuda")
assert np.abs(K.softmax(x).cpu().numpy() - O.softmax_rows_f64(x.cpu().numpy())).max() < 1e-5
from paper_2505_08091_b200 import nw as NW  # noqa: E402
from nw_perms import rotate_cells, skew_order, xor_cells  # noqa: E402
n = 300
sim = np.random.default_rng(3).integers(-10, 11, size=(n, n), dtype=np.int32)
for lay in (NW.nw_layout(n, tile_rows=64, tile_order=skew_order(5, 3), cell_order=xor_cells(64)),
            NW.nw_layout(n, tile_rows=96, tile_order="col", cell_order=rotate_cells(96))):
    assert np.array_equal(K.nw_score(torch.from_numpy(sim).cuda(), 10, layout=lay).cpu().numpy(), O.nw(sim, 10))
import ctypes  # noqa: E402
import test_template as TT  # noqa: E402
mod = K.compile_template(TT.USER_TEMPLATE, TT.USER_MANIFEST)
src = torch.arange(256 * 256, dtype=torch.float32, device="cuda")
dst = torch.empty_like(src)
mod.launch("lego_tpl_tile", (256,), (256,), [ctypes.c_void_p(src.data_ptr()), ctypes.c_void_p(dst.data_ptr())])
assert np.array_equal(dst.cpu().numpy(), O.remap(src.cpu().numpy(), None, O.parse(
    "GroupBy([256,256]).OrderBy(RegP([8,32,8,32],[1,3,2,4]))")))
torch.cuda.synchronize()
print("sanitize driver: all checks passed;", len(plans), "remap plans:", sorted(set(p.split(",")[0] for p in plans)))
