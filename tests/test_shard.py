"""Multi-process host logic of the sharding layer: world_size 2 over gloo on
CPU, with the per-shard compute injected (the GPU kernel is replaced by the
scalar layout API, itself pinned to the reference by test_frontend.py)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2505_08091_b200 as L
from paper_2505_08091_b200 import shard


def cpu_remap(x, src_layout, dst_layout):
    """dst[dst.apply(v)] = src[src.apply(v)] with the scalar API (tiny sizes)."""
    some = src_layout or dst_layout
    dims = some.dims
    n = int(np.prod(dims))
    flat = x.reshape(-1, n)
    out = torch.empty_like(flat)
    for v in range(n):
        idx = []
        rem = v
        for d in reversed(dims):
            idx.append(rem % d)
            rem //= d
        idx = tuple(reversed(idx))
        s = src_layout.apply(idx) if src_layout is not None else v
        t = dst_layout.apply(idx) if dst_layout is not None else v
        out[:, t] = flat[:, s]
    return out.reshape(x.shape[:-1] + (n,)) if x.dim() > 1 else out.reshape(n)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, fn, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        fn(rank, world)
        q.put((rank, None))
    except Exception as exc:  # noqa: BLE001
        import traceback
        q.put((rank, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


def run_world(fn, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, fn, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    errs = [e for _, e in results if e]
    assert not errs, errs[0]


def _batch_case(rank, world):
    g = L.parse_layout("GroupBy([8,8]).OrderBy(Col(8,8))")
    x = torch.arange(5 * 64, dtype=torch.int32).reshape(5, 64)        # 5 items: ragged over 2
    out = shard.sharded(cpu_remap, x, None, g, gather=True)
    want = cpu_remap(x, None, g)
    assert torch.equal(out, want)
    p = shard.plan(5)
    assert (p.start, p.stop) == ((0, 3) if rank == 0 else (3, 5))


def _transpose_case(rank, world):
    n_rows, n_cols = 8, 12
    full = torch.arange(n_rows * n_cols, dtype=torch.int32).reshape(n_rows, n_cols)
    R = n_rows // world
    local = full[rank * R:(rank + 1) * R].contiguous()
    got = shard.transpose_rows(local, n_rows, n_cols, compute=cpu_remap)
    C = n_cols // world
    assert torch.equal(got, full.t()[rank * C:(rank + 1) * C])
    # and it is exactly the LEGO Col layout of the whole matrix
    g = L.parse_layout(f"GroupBy([{n_rows},{n_cols}]).OrderBy(Col({n_cols},{n_rows}))")
    whole = cpu_remap(full.reshape(-1), None, g).reshape(n_cols, n_rows)
    assert torch.equal(got, whole[rank * C:(rank + 1) * C])


def test_batch_sharding_with_ragged_gather():
    run_world(_batch_case)


def test_row_sharded_transpose_all_to_all():
    run_world(_transpose_case)


def test_plan_covers_everything():
    for total in (0, 1, 7, 8, 65537):
        for world in (1, 2, 4, 8):
            spans = [shard.ShardPlan(total, world, r) for r in range(world)]
            covered = sum(p.count for p in spans)
            assert covered == total
            assert all(a.stop == b.start for a, b in zip(spans, spans[1:]))


def test_single_process_defaults():
    x = torch.arange(16).reshape(4, 4)
    assert shard.plan(4).count == 4
    assert torch.equal(shard.local_slice(x), x)


@pytest.mark.parametrize("world,R,C", [(2, 16, 8), (4, 8, 16), (8, 32, 8)])
def test_fused_transpose_routing_every_rank(world, R, C):
    """transpose_rows_fused's routing, evaluated for every rank and every
    destination element: the union of all ranks' routed stores is exactly
    the transposed matrix, sharded by rows, each element written once."""
    from paper_2505_08091_b200 import lower, staging
    from paper_2505_08091_b200.expr import Var, VarRange
    n_rows, n_cols = world * R, world * C
    full = np.arange(n_rows * n_cols, dtype=np.int64).reshape(n_rows, n_cols)
    shards = np.full((world, C * n_rows), -1, dtype=np.int64)
    for rank in range(world):
        layout, route = shard.fused_transpose_route(R, C, world, rank)
        f, g, n_dst, n_src = lower.gather_expr(None, layout)
        assert (n_dst, n_src) == (R * n_cols, R * n_cols)
        v = np.arange(n_dst)
        src_idx = staging.eval_vec(g, {"f": v})                 # local source element of v
        peer_e, off_e = route.fn(f)
        peer = staging.eval_vec(lower.as_expr(peer_e), {"f": v})
        off = staging.eval_vec(lower.as_expr(off_e), {"f": v})
        local = full[rank * R:(rank + 1) * R].reshape(-1)
        assert np.all(shards[peer, off] == -1)
        shards[peer, off] = local[src_idx]
    want = full.T.reshape(world, C * n_rows)
    np.testing.assert_array_equal(shards, want)


def test_fused_transpose_plan_proves_vector_routing():
    """The planner accepts the routing (16-byte vectors stay in one peer,
    contiguous, aligned) and picks the routed register transpose."""
    from paper_2505_08091_b200 import kernels, runtime
    layout, route = shard.fused_transpose_route(256, 128, 4, 1)
    for elem in (2, 4):
        p = kernels.plan_remap(None, layout, elem, route)
        assert p.kind == runtime.KIND_TRANSPOSE and "routed over 4 peers" in p.detail
    # a routing that splits vectors across peers is refused
    bad = kernels.Route(2, lambda v: (v % 2, v // 2), ("bad",))
    with pytest.raises(L.UnsupportedNode):
        kernels.plan_remap(None, layout, 4, bad)


def test_nw_bands_cover_the_strips_in_order():
    from paper_2505_08091_b200 import shard
    for n, world in ((16384, 8), (16384, 3), (300, 4), (100, 2), (1, 1), (129, 2)):
        bands = shard.nw_bands(n, world)
        nc = -(-n // 128)
        assert len(bands) == world and bands[0][0] == 0 and bands[-1][1] == nc
        assert all(b0[1] == b1[0] for b0, b1 in zip(bands, bands[1:]))
        assert all(e >= b for b, e in bands)



def cpu_map(layout, first, count):
    """layout.apply over logical indices first .. first+count-1 (scalar API)."""
    dims = layout.dims
    out = []
    for v in range(first, first + count):
        idx, rem = [], v
        for d in reversed(dims):
            idx.append(rem % d)
            rem //= d
        out.append(layout.apply(tuple(reversed(idx))))
    return torch.tensor(out, dtype=torch.int64)


def _remap_sharded_case(rank, world):
    for dsl in ("GroupBy([8,8]).OrderBy(GenP([8,8], antidiag))",
                "GroupBy([6,10]).OrderBy(RegP([2,3,2,5],[3,1,4,2]))",
                "GroupBy([7,9]).OrderBy(Col(9,7))"):
        g = L.parse_layout(dsl)
        n = int(np.prod(g.dims))
        full = (torch.arange(n, dtype=torch.int32) * 7 + 3)
        lp = -(-n // world)
        local = full[min(n, rank * lp):min(n, (rank + 1) * lp)]
        got = shard.remap_sharded(local, g, compute_map=cpu_map)
        whole = cpu_remap(full, None, g)
        assert torch.equal(got, whole[min(n, rank * lp):min(n, (rank + 1) * lp)]), dsl


@pytest.mark.parametrize("world", [2, 3])
def test_remap_sharded_any_bijective_layout(world):
    run_world(_remap_sharded_case, world=world)


def _gather_bands_case(rank, world):
    n = 300                                     # 3 strips over 4 ranks: the last band is empty
    bands = shard.nw_bands(n, world)
    whole = torch.arange((n + 1) * (n + 1), dtype=torch.int32).reshape(n + 1, n + 1)
    b0, e0 = bands[rank]
    out = torch.full_like(whole, -1)
    out[0, :] = whole[0, :]
    out[:, 0] = whole[:, 0]
    lo, hi = 1 + 128 * b0, min(n, 128 * e0) + 1
    if hi > lo:
        out[:, lo:hi] = whole[:, lo:hi]
    assert torch.equal(shard.gather_nw_bands(out, bands), whole)


def test_gather_nw_bands_with_an_empty_band():
    run_world(_gather_bands_case, world=4)
