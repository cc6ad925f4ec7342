"""Multi-GPU sharding of independent layout work (one process per GPU).

The LEGO hot path is embarrassingly parallel over independent matrices (a
batch) and, for row-local kernels, over rows: every shard is processed by
its own GPU with no data-path collective.  NCCL appears only where a result
has to cross shards:

* :func:`gather_shards` -- reassemble a batch-sharded result on every rank
  (``all_gather_into_tensor``; ragged shards are padded and trimmed);
* :func:`transpose_rows` -- a *single* matrix whose rows are split across
  ranks, remapped into a layout that needs other ranks' rows (the
  column-major ``Col`` layout): one ``all_to_all_single`` of row-block x
  column-block tiles, then each rank finishes with local LEGO remaps;
* :func:`transpose_rows_fused` -- the same result as one routed transpose
  kernel per rank that stores straight into the other ranks' shards through
  NVLink peer memory (torch symmetric memory), no NCCL in the data path;
* :func:`remap_sharded` -- any bijective layout over one array split across
  ranks (destination positions by the GPU map, one uneven all-to-all);
* :class:`NwBanded` -- one Needleman-Wunsch alignment split by column bands,
  the wavefront kernel of each band polling the previous band's edge column
  in the peer GPU's memory (the hand-off inside the kernel).

All functions take ``compute=`` so the host logic is testable on CPU with
the ``gloo`` backend (tests/test_shard.py injects the oracle); the default
compute is the GPU kernel of :mod:`.kernels`.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Callable, Optional

from .errors import ShapeMismatch


@dataclass(frozen=True)
class ShardPlan:
    """Contiguous split of ``total`` independent items over ``world`` ranks."""

    total: int
    world: int
    rank: int

    @property
    def per_rank(self) -> int:
        return math.ceil(self.total / self.world) if self.world else 0

    @property
    def start(self) -> int:
        return min(self.total, self.rank * self.per_rank)

    @property
    def stop(self) -> int:
        return min(self.total, self.start + self.per_rank)

    @property
    def count(self) -> int:
        return self.stop - self.start

    def bounds(self, rank: int):
        return ShardPlan(self.total, self.world, rank).start, ShardPlan(self.total, self.world, rank).stop


def _dist():
    import torch.distributed as dist
    return dist


def world_and_rank(group=None):
    dist = _dist()
    if not dist.is_available() or not dist.is_initialized():
        return 1, 0
    return dist.get_world_size(group), dist.get_rank(group)


def plan(total: int, group=None) -> ShardPlan:
    world, rank = world_and_rank(group)
    return ShardPlan(total, world, rank)


def local_slice(x, group=None):
    """This rank's contiguous share of the leading (batch) dimension of x."""
    p = plan(x.shape[0], group)
    return x[p.start:p.stop]


def sharded(fn: Callable, x, *args, group=None, gather: bool = False, **kw):
    """Apply ``fn`` (e.g. ``kernels.remap``) to this rank's batch shard; with
    ``gather=True`` return the full result on every rank."""
    p = plan(x.shape[0], group)
    out = fn(x[p.start:p.stop], *args, **kw)
    return gather_shards(out, p, group) if gather else out


def gather_shards(local, p: ShardPlan, group=None):
    """All-gather equally-padded batch shards and trim to ``p.total``."""
    import torch
    dist = _dist()
    if p.world == 1:
        return local
    pad = p.per_rank - local.shape[0]
    if pad:
        local = torch.cat([local, local.new_zeros((pad,) + tuple(local.shape[1:]))])
    full = local.new_empty((p.per_rank * p.world,) + tuple(local.shape[1:]))
    if hasattr(dist, "all_gather_into_tensor") and local.is_cuda:
        dist.all_gather_into_tensor(full, local.contiguous(), group=group)
    else:
        parts = list(full.chunk(p.world))
        dist.all_gather(parts, local.contiguous(), group=group)
        full = torch.cat(parts)
    return full[:p.total]


def nw_bands(n: int, world: int):
    """Strip ranges [begin, end) (128-column strips) of an n x n NW per rank:
    contiguous, as even as whole strips allow (ranks past the last strip get
    an empty band)."""
    nc = -(-n // 128)
    per = -(-nc // world) if world else 0
    return [(min(nc, r * per), min(nc, (r + 1) * per)) for r in range(world)]


class NwBanded:
    """One Needleman-Wunsch alignment (or a batch) split by column bands over
    the ranks, set up once (symmetric edge buffer, peer view) and run per call.

    Rank r computes strips ``nw_bands(n, world)[r]`` of every matrix with the
    wavefront kernel, reading the previous band's edge column straight from
    rank r-1's memory over NVLink (torch symmetric memory, system-scope
    sentinel words): the hand-off is inside the kernel, no NCCL on the data
    path; the band's own right edge lands in its symmetric buffer for rank
    r+1.  Each call presets the edge words, device-barriers, runs the band and
    device-barriers again (the next band has read the edge), all on the
    current stream.  SURVEY.md 8(e): the NW row's "next" item."""

    def __init__(self, n: int, batch: int, device, *, group=None, max_ctas: int = 0):
        import torch
        from torch.distributed import _symmetric_memory as symm
        from . import kernels
        dist = _dist()
        self.world, self.rank = world_and_rank(group)
        self.n, self.batch, self.group, self.max_ctas = n, batch, group, max_ctas
        self.bands = nw_bands(n, self.world)
        self.begin, self.end = self.bands[self.rank]
        strips_max = max(e - b for b, e in self.bands)
        self.bnd = symm.empty(max(1, kernels.nw_band_words(n, strips_max, batch)), dtype=torch.int32, device=device)
        self.handle = symm.rendezvous(self.bnd, group if group is not None else dist.group.WORLD)
        self.left, self.left_strips = None, 0
        if self.begin > 0:
            pb, pe = self.bands[self.rank - 1]
            self.left = self.handle.get_buffer(self.rank - 1, (self.bnd.numel(),), torch.int32)
            self.left_strips = pe - pb

    def __call__(self, sim, penalty: int, *, out=None, gather: bool = False):
        import torch
        from . import kernels
        n = self.n
        if sim.shape[-1] != n or sim.numel() != self.batch * n * n:
            raise ShapeMismatch(f"sim {tuple(sim.shape)} does not match the banded plan ({self.batch} x {n} x {n})")
        if out is None:
            out = torch.empty(*sim.shape[:-2], n + 1, n + 1, dtype=torch.int32, device=sim.device)
        self.bnd.fill_(kernels.NW_EMPTY_WORD)
        self.handle.barrier(channel=0)          # every band's edge words are preset before any band runs
        if self.end > self.begin:
            kernels.nw_score_band(sim, penalty, (self.begin, self.end), self.bnd, left=self.left,
                                  left_strips=self.left_strips, out=out, max_ctas=self.max_ctas)
        else:                                   # no strip for this rank: borders only
            edge = -torch.arange(n + 1, device=sim.device, dtype=torch.int32) * int(penalty)
            out[..., 0, :] = edge
            out[..., :, 0] = edge
        self.handle.barrier(channel=0)          # the next band has read this band's edge
        if not gather or self.world == 1:
            return out
        return gather_nw_bands(out, self.bands, group=self.group)


def nw_score_banded(sim, penalty: int, *, group=None, gather: bool = True, max_ctas: int = 0):
    """:class:`NwBanded` for one call: every rank passes the (replicated)
    ``sim``; with ``gather=True`` every rank returns the full score (bands
    all-gathered), else the full-size score with only this rank's columns
    (and the borders) written."""
    batch = 1
    for d in sim.shape[:-2]:
        batch *= d
    return NwBanded(sim.shape[-1], batch, sim.device, group=group, max_ctas=max_ctas)(sim, penalty, gather=gather)


def gather_nw_bands(out, bands, *, group=None):
    """All-gather the column bands of full-size NW scores (each rank's
    ``out`` holds its band's columns 1 + 128*begin .. 128*end, plus the borders)."""
    import torch
    dist = _dist()
    n = out.shape[-1] - 1
    w = 128 * max(e - b for b, e in bands)
    lead = out.shape[:-2]
    rank = world_and_rank(group)[1]
    b0, e0 = bands[rank]
    c0, c1 = 1 + 128 * b0, min(n, 128 * e0) + 1
    mine = out.new_zeros(*lead, n + 1, w)
    if c1 > c0:                                 # ranks past the last strip hold no columns
        mine[..., :, :c1 - c0] = out[..., :, c0:c1]
    parts = [torch.empty_like(mine) for _ in bands]
    dist.all_gather(parts, mine.contiguous(), group=group)
    full = out.clone()
    for (b, e), part in zip(bands, parts):
        lo, hi = 1 + 128 * b, min(n, 128 * e) + 1
        if hi > lo:
            full[..., :, lo:hi] = part[..., :, :hi - lo]
    return full


def transpose_rows(local_rows, n_rows: int, n_cols: int, *, group=None,
                   compute: Optional[Callable] = None):
    """Distributed ``Col`` layout of one row-sharded matrix.

    Rank r holds rows [r*R, (r+1)*R) of an (n_rows x n_cols) row-major
    matrix (R = n_rows / world).  The result in the layout
    ``GroupBy([n_rows, n_cols]).OrderBy(Col(n_cols, n_rows))`` is the
    transposed matrix; rank r returns its rows [r*C, (r+1)*C) of that
    (n_cols x n_rows) array (C = n_cols / world).

    Step 1 (local, LEGO): cut the local rows into ``world`` column blocks,
    each a contiguous (R x C) tile -- a batched tile_by remap.
    Step 2 (NCCL): one ``all_to_all_single`` so rank r receives tile r of
    every rank.  Step 3 (local, LEGO): transpose each received (R x C) tile
    to (C x R) and lay the tiles side by side.
    """
    import torch
    dist = _dist()
    world, rank = world_and_rank(group)
    if n_rows % world or n_cols % world:
        raise ShapeMismatch(f"{n_rows}x{n_cols} does not split over {world} ranks")
    R, C = n_rows // world, n_cols // world
    if local_rows.shape != (R, n_cols):
        raise ShapeMismatch(f"local rows {tuple(local_rows.shape)} != {(R, n_cols)}")
    tile_layout, t_layout = _transpose_layouts(R, C, world)
    run = compute or _gpu_remap
    # (R, world*C) row-major -> world tiles of (R, C), contiguous per tile
    tiles = run(local_rows.reshape(-1), None, tile_layout).reshape(world, R * C)
    recv = torch.empty_like(tiles)
    if world > 1:
        dist.all_to_all_single(recv, tiles, group=group)
    else:
        recv.copy_(tiles)
    # recv[q] is tile (rows of rank q) x (my column block): transpose each to (C, R)
    tt = run(recv, None, t_layout)                          # (world, C*R), each C x R
    # place tiles side by side: out[c, q*R + r] = tt[q, c*R + r]
    return run(tt.reshape(-1), None, _sidebyside_layout(R, C, world)).reshape(C, world * R)


def remap_sharded(local, layout, *, group=None, compute_map: Optional[Callable] = None):
    """Any bijective layout applied to ONE array split over the ranks.

    Rank r holds the logical elements [r*Lp, (r+1)*Lp) (row-major logical
    index, Lp = ceil(N / world)); it returns its share [r*Pp, (r+1)*Pp) of the
    physical result ``y[layout.apply(v)] = x[v]`` (Pp = ceil(N / world)).

    Step 1 (local, LEGO): the destination positions of the local range --
    ``kernels.apply_map(layout, first=, count=)`` on the GPU.  Step 2: bucket
    the elements by owning rank and exchange values and in-shard offsets with
    two ``all_to_all_single`` calls (uneven splits).  Step 3 (local): place the
    received values.  The generic path of SURVEY.md 8(e) for single-matrix
    layouts that are not digit permutations (e.g. cfg4a's anti-diagonal
    GenP); ``compute_map(layout, first, count)`` replaces the GPU map in CPU
    tests."""
    import torch
    from . import lower
    dist = _dist()
    world, rank = world_and_rank(group)
    n = lower.logical_size(layout)
    if lower.physical_size(layout) != n or getattr(layout, "injective", False):
        raise ShapeMismatch("remap_sharded needs a bijective layout (logical size == physical size)")
    lp = -(-n // world)
    start = min(n, rank * lp)
    count = min(n, start + lp) - start
    flat = local.reshape(-1)
    if flat.numel() != count:
        raise ShapeMismatch(f"rank {rank} holds {flat.numel()} elements, expected {count} of {n}")
    if compute_map is None:
        from . import kernels
        pos = kernels.apply_map(layout, dtype=torch.int64, device=flat.device, first=start, count=count)
    else:
        pos = compute_map(layout, start, count).to(flat.device)
    pos = pos.to(torch.int64)
    owner = torch.div(pos, lp, rounding_mode="floor")
    order = torch.argsort(owner, stable=True)
    vals = flat[order].contiguous()
    offs = (pos - owner * lp)[order].contiguous()
    send = torch.bincount(owner, minlength=world).to(torch.int64)
    recv = torch.empty_like(send)
    if world > 1:
        dist.all_to_all_single(recv, send, group=group)
    else:
        recv.copy_(send)
    sc, rc = [int(v) for v in send.tolist()], [int(v) for v in recv.tolist()]
    rvals = flat.new_empty(sum(rc))
    roffs = torch.empty(sum(rc), dtype=torch.int64, device=flat.device)
    if world > 1:
        dist.all_to_all_single(rvals, vals, rc, sc, group=group)
        dist.all_to_all_single(roffs, offs, rc, sc, group=group)
    else:
        rvals.copy_(vals)
        roffs.copy_(offs)
    mine = min(n, (rank + 1) * lp) - min(n, rank * lp)
    if sum(rc) != mine:
        raise ShapeMismatch(f"rank {rank} received {sum(rc)} elements for {mine} positions (layout not bijective?)")
    out = flat.new_empty(mine)
    out[roffs] = rvals
    return out


def transpose_rows_fused(local_rows, n_rows: int, n_cols: int, *, group=None):
    """:func:`transpose_rows` as ONE kernel per rank (B200/NVSwitch path).

    Rank r's output shard lives in torch symmetric memory, so every rank can
    store into every other rank's shard over NVLink.  Each rank runs one
    routed register transpose of its local rows (``kernels.remap_routed``):
    the 16-byte vectors of transposed row c go straight to rank c // C, at
    the column offset of the sending rank's rows -- no staging tiles, no
    NCCL all-to-all, the exchange overlaps the transpose tile by tile.  Two
    device-side barriers order it: every shard is free before anyone
    writes, and every store has landed before anyone reads.  Same result as
    :func:`transpose_rows` (tests/test_shard.py checks the routing for every
    rank on CPU; tests/test_gpu_kernels.py runs the routed kernel on a GPU
    against per-rank buffers).  Repeated calls should hold one
    :class:`FusedTranspose` (the symmetric buffer is set up once)."""
    world, _rank = world_and_rank(group)
    if n_rows % world or n_cols % world:
        raise ShapeMismatch(f"{n_rows}x{n_cols} does not split over {world} ranks")
    ft = FusedTranspose(n_rows, n_cols, local_rows.dtype, local_rows.device, group=group)
    return ft(local_rows)


class FusedTranspose:
    """Set-up of :func:`transpose_rows_fused` kept across calls: the
    symmetric output shard, its peer address table and the routed program."""

    def __init__(self, n_rows: int, n_cols: int, dtype, device, *, group=None):
        import torch
        from torch.distributed import _symmetric_memory as symm
        dist = _dist()
        world, rank = world_and_rank(group)
        if n_rows % world or n_cols % world:
            raise ShapeMismatch(f"{n_rows}x{n_cols} does not split over {world} ranks")
        self.R, self.C, self.world, self.rank = n_rows // world, n_cols // world, world, rank
        self.n_rows, self.n_cols = n_rows, n_cols
        self.out = symm.empty((self.C, n_rows), dtype=dtype, device=device)
        self.handle = symm.rendezvous(self.out, group if group is not None else dist.group.WORLD)
        self.peers = torch.tensor([int(p) for p in self.handle.buffer_ptrs], dtype=torch.int64, device=device)
        self.layout, self.route = fused_transpose_route(self.R, self.C, world, rank)

    def __call__(self, local_rows):
        from . import kernels
        if local_rows.shape != (self.R, self.n_cols):
            raise ShapeMismatch(f"local rows {tuple(local_rows.shape)} != {(self.R, self.n_cols)}")
        self.handle.barrier(channel=0)
        kernels.remap_routed(local_rows.reshape(-1), None, self.layout, self.peers, self.route)
        self.handle.barrier(channel=0)
        return self.out


def fused_transpose_route(R: int, C: int, world: int, rank: int):
    """(local layout, kernels.Route) of :func:`transpose_rows_fused` on
    ``rank``: the local (R x world*C) rows transposed to (world*C x R)
    (position v = c*R + r), and v routed to rank c // C at element offset
    (c % C) * (world*R) + rank*R + r of that rank's (C x world*R) shard."""
    from .kernels import Route
    from .layout import GroupBy, RegP
    n_cols, n_rows = world * C, world * R
    layout = GroupBy([R, n_cols]).order_by(RegP((R, n_cols), (2, 1)))

    def fn(v):
        c, r = v // R, v % R
        return c // C, (c % C) * n_rows + rank * R + r

    return layout, Route(world, fn, ("transpose_rows", R, C, world, rank))


def _transpose_layouts(R, C, world):
    from .layout import GroupBy, RegP
    # logical (r, q, c) of the local (R, world*C) rows -> position q*R*C + r*C + c
    tile = GroupBy([R, world, C]).order_by(RegP((R, world, C), (2, 1, 3)))
    # logical (r, c) of an R x C tile -> position c*R + r (column-major)
    trans = GroupBy([R, C]).order_by(RegP((R, C), (2, 1)))
    return tile, trans


def _sidebyside_layout(R, C, world):
    from .layout import GroupBy, RegP
    # logical (q, c, r) of `world` stacked C x R tiles -> position c*world*R + q*R + r
    return GroupBy([world, C, R]).order_by(RegP((world, C, R), (2, 1, 3)))


def _gpu_remap(x, src_layout, dst_layout):
    from . import kernels
    return kernels.remap(x, src_layout, dst_layout)
