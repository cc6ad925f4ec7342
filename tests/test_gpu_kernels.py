"""Fixed kernels on the GPU: tcgen05 GEMM (max-rel <= 1e-2 vs fp32/fp64),
row softmax (<= 1e-5 vs float64), Needleman-Wunsch (bit-exact vs the C DP)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2505_08091_b200 import kernels as K  # noqa: E402
from oracle import oracle as O  # noqa: E402


def _gemm_check(M, N, Kd, batch=1, raster=1, seed=5):
    g = torch.Generator(device="cuda").manual_seed(seed)
    a = torch.randn(batch, M, Kd, device="cuda", generator=g).to(torch.bfloat16)
    b = torch.randn(batch, N, Kd, device="cuda", generator=g).to(torch.bfloat16)
    c = K.gemm(a, b, raster=raster)
    ref = torch.matmul(a.double(), b.double().transpose(-1, -2))
    err = (c.double() - ref).abs()
    # max-rel with the tolerance of north_star: |C - ref| / max(|ref|, 1e-2 * max|ref|)
    denom = torch.clamp(ref.abs(), min=1e-2 * ref.abs().max().item())
    rel = (err / denom).max().item()
    assert rel <= 1e-2, (M, N, Kd, batch, rel)
    return rel


def test_gemm_small_shapes():
    # kernel selection by shape (csrc/gemm_tcgen05.cu): M % 256 and N % 512 -> CTA-pair 256x512
    # tiles; M % 256 and N % 256 -> CTA-pair 256x256; otherwise single-CTA 128x256
    _gemm_check(128, 256, 64)                   # single CTA
    _gemm_check(256, 512, 128, batch=2)         # pair, 256x512
    _gemm_check(384, 256, 1024, raster=0)       # single CTA
    _gemm_check(2048, 1024, 512, batch=3)       # pair, 256x512
    _gemm_check(512, 768, 256, raster=4)        # pair, 256x256
    _gemm_check(1024, 1280, 192, batch=2)       # pair, 256x256 (N % 512 = 256)


@pytest.mark.parametrize("M,N,Kd,batch", [(8, 8, 8, 1), (100, 72, 40, 1), (257, 520, 136, 2),
                                          (1000, 1000, 1000, 1), (130, 264, 72, 3)])
def test_gemm_ragged_shapes(M, N, Kd, batch):
    # tails: TMA zero-fills operand boxes past M, N, K; the epilogue masks rows >= M, cols >= N
    _gemm_check(M, N, Kd, batch=batch)


def test_gemm_8192_cubed():
    _gemm_check(8192, 8192, 8192)


@pytest.mark.parametrize("rows,cols", [(3, 1), (5, 7), (17, 1023), (2, 4097), (4, 300001)])
def test_softmax_ragged_rows(rows, cols):
    """cols % 4 != 0 takes the scalar kernel (max-rel <= 1e-5 vs float64)."""
    g = torch.Generator(device="cuda").manual_seed(cols)
    x = torch.randn(rows, cols, device="cuda", generator=g) * 4
    y = K.softmax(x)
    ref = torch.softmax(x.double(), dim=-1)
    rel = ((y.double() - ref).abs() / ref.abs().clamp_min(1e-30)).max().item()
    assert rel <= 1e-5, rel


def test_gemm_rejects_bad_shapes():
    import paper_2505_08091_b200 as L
    a = torch.zeros(100, 60, device="cuda", dtype=torch.bfloat16)      # K % 8 != 0
    with pytest.raises(L.ShapeMismatch):
        K.gemm(a, a)


@pytest.mark.parametrize("n", [1, 7, 64, 100, 257, 1024])
def test_nw_vs_c_dp(n):
    rng = np.random.default_rng(n)
    sim = rng.integers(-10, 11, size=(2, n, n), dtype=np.int32)
    got = K.nw_score(torch.from_numpy(sim).cuda(), 10).cpu().numpy()
    for b in range(2):
        np.testing.assert_array_equal(got[b], O.nw(sim[b], 10))


@pytest.mark.parametrize("p", [0, -2, 37])
def test_nw_penalties_and_wide_scores(p):
    """The library strip kernel with zero, negative and large penalties, and
    similarities up to +-2^20 (scores near the kernel's +-2^30 contract)."""
    rng = np.random.default_rng(100 + p)
    n = 333
    sim = rng.integers(-(1 << 20), 1 << 20, size=(2, n, n), dtype=np.int32)
    sim[1] = rng.integers(-3, 4, size=(n, n), dtype=np.int32)
    got = K.nw_score(torch.from_numpy(sim).cuda(), p).cpu().numpy()
    for b in range(2):
        np.testing.assert_array_equal(got[b], O.nw(sim[b], p))


def test_nw_strips_more_than_ctas():
    """158 strips on 148 persistent CTAs: CTAs claim a second strip (ticket
    order across the batch), n not a multiple of 4 (scalar sim staging)."""
    rng = np.random.default_rng(9)
    n = 10001
    sim = rng.integers(-10, 11, size=(2, n, n), dtype=np.int32)
    got = K.nw_score(torch.from_numpy(sim).cuda(), 7).cpu().numpy()
    for b in range(2):
        np.testing.assert_array_equal(got[b], O.nw(sim[b], 7))


def test_nw_16384():
    rng = np.random.default_rng(4)
    n = 16384
    sim = rng.integers(-10, 11, size=(n, n), dtype=np.int32)
    got = K.nw_score(torch.from_numpy(sim).cuda(), 10).cpu().numpy()
    np.testing.assert_array_equal(got, O.nw(sim, 10))


def test_empty_inputs():
    """Empty batches and zero-size problems return empty results without launching."""
    import paper_2505_08091_b200 as L
    g = L.parse_layout("GroupBy([64,64]).OrderBy(Col(64,64))")
    x = torch.empty(0, 64 * 64, device="cuda", dtype=torch.float32)
    assert K.remap(x, None, g).shape == (0, 64 * 64)
    assert K.softmax(torch.empty(0, 8, device="cuda")).shape == (0, 8)
    assert K.softmax(torch.empty(5, 0, device="cuda")).shape == (5, 0)
    s = K.nw_score(torch.empty(0, 5, 5, device="cuda", dtype=torch.int32), 10)
    assert s.shape == (0, 6, 6)
    s = K.nw_score(torch.empty(0, 0, device="cuda", dtype=torch.int32), 10)
    assert s.shape == (1, 1) and s.item() == 0
    c = K.gemm(torch.empty(0, 128, 64, device="cuda", dtype=torch.bfloat16),
               torch.empty(0, 256, 64, device="cuda", dtype=torch.bfloat16))
    assert c.shape == (0, 128, 256)


@pytest.mark.parametrize("a_layout", ["row", "col"])
@pytest.mark.parametrize("b_layout", ["row", "col"])
@pytest.mark.parametrize("M,N,Kd,batch", [(256, 512, 128, 1), (512, 768, 320, 2), (136, 264, 72, 1),
                                          (2048, 2048, 2048, 1)])
def test_matmul_four_data_layouts(a_layout, b_layout, M, N, Kd, batch):
    """The paper's four matmul variants (Row/Col data layout of A and B,
    PAPER.md:1226-1227): MN-major operands go to tcgen05 directly."""
    g = torch.Generator(device="cuda").manual_seed(M + N + Kd)
    A = torch.randn(batch, M, Kd, device="cuda", generator=g).to(torch.bfloat16)
    B = torch.randn(batch, Kd, N, device="cuda", generator=g).to(torch.bfloat16)
    a = A if a_layout == "row" else A.transpose(-1, -2).contiguous()      # Col: stored column-major
    b = B if b_layout == "row" else B.transpose(-1, -2).contiguous()
    c = K.matmul(a, b, a_layout=a_layout, b_layout=b_layout)
    ref = torch.matmul(A.double(), B.double())
    denom = torch.clamp(ref.abs(), min=1e-2 * ref.abs().max().item())
    rel = ((c.double() - ref).abs() / denom).max().item()
    assert rel <= 1e-2, (a_layout, b_layout, M, N, Kd, rel)


@pytest.mark.parametrize("dtype", [torch.int8, torch.int16, torch.int32, torch.int64])
@pytest.mark.parametrize("world,R,C", [(4, 256, 128), (2, 64, 512)])
def test_routed_transpose_into_peer_buffers(dtype, world, R, C):
    """The fused remap + all-to-all kernel of shard.transpose_rows_fused, with
    the `world` ranks' output shards emulated as separate buffers on one GPU:
    every rank's routed transpose stores into all shards; together they hold
    the transposed matrix, sharded by rows."""
    from paper_2505_08091_b200 import shard
    n_rows, n_cols = world * R, world * C
    full = (torch.arange(n_rows * n_cols, device="cuda", dtype=torch.int64) * 2654435761 % 1000003)
    full = full.to(dtype).reshape(n_rows, n_cols)
    shards = [torch.full((C, n_rows), -1, dtype=dtype, device="cuda") for _ in range(world)]
    peers = torch.tensor([t.data_ptr() for t in shards], dtype=torch.int64, device="cuda")
    for rank in range(world):
        layout, route = shard.fused_transpose_route(R, C, world, rank)
        K.remap_routed(full[rank * R:(rank + 1) * R].reshape(-1), None, layout, peers, route)
    torch.cuda.synchronize()
    want = full.t().contiguous()
    for q in range(world):
        assert torch.equal(shards[q], want[q * C:(q + 1) * C]), q


def test_transpose_rows_fused_single_rank_symmetric_memory(tmp_path):
    """transpose_rows_fused end to end through torch symmetric memory on a
    one-rank NCCL group (the only multi-process shape one GPU allows)."""
    import torch.distributed as dist
    from paper_2505_08091_b200 import shard
    if dist.is_initialized():
        pytest.skip("a process group is already initialised")
    try:
        dist.init_process_group("nccl", init_method=f"file://{tmp_path}/pg", world_size=1, rank=0,
                                device_id=torch.device("cuda:0"))
    except Exception as exc:  # noqa: BLE001
        pytest.skip(f"NCCL process group unavailable: {exc}")
    try:
        x = torch.randint(-1000, 1000, (512, 1024), device="cuda", dtype=torch.int32)
        try:
            out = shard.transpose_rows_fused(x, 512, 1024)
        except (RuntimeError, NotImplementedError) as exc:
            pytest.skip(f"symmetric memory unavailable: {exc}")
        torch.cuda.synchronize()
        assert torch.equal(out, x.t())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n,nbands,batch,reverse", [(1000, 2, 1, False), (1000, 3, 2, True), (4100, 4, 1, True),
                                                    (16384, 2, 1, False), (300, 4, 1, False)])
def test_nw_column_bands_match_the_whole(n, nbands, batch, reverse):
    """The multi-GPU single-alignment path (shard.nw_score_banded) on one GPU:
    each band on its own stream with its own edge buffer, band r polling band
    r-1's edge column (system scope), bands launched in either order and
    running concurrently (max_ctas splits the SMs); assembled result
    bit-exact against the C DP."""
    from paper_2505_08091_b200 import shard
    rng = np.random.default_rng(n + nbands)
    sim = rng.integers(-10, 11, size=(batch, n, n), dtype=np.int32)
    dsim = torch.from_numpy(sim).cuda()
    bands = shard.nw_bands(n, nbands)
    bnds = [torch.full((max(1, K.nw_band_words(n, e - b, batch)),), K.NW_EMPTY_WORD, dtype=torch.int32,
                       device="cuda") for b, e in bands]
    outs = [torch.zeros(batch, n + 1, n + 1, dtype=torch.int32, device="cuda") for _ in bands]
    streams = [torch.cuda.Stream() for _ in bands]
    torch.cuda.synchronize()
    cap = 148 // nbands
    for r in (range(nbands)[::-1] if reverse else range(nbands)):
        b, e = bands[r]
        if e == b:
            continue
        pb, pe = bands[r - 1] if r else (0, 0)
        with torch.cuda.stream(streams[r]):
            K.nw_score_band(dsim, 10, (b, e), bnds[r], left=bnds[r - 1] if b else None, left_strips=pe - pb,
                            out=outs[r], max_ctas=cap, stream=streams[r])
    torch.cuda.synchronize()
    full = outs[0].clone()
    for (b, e), o in zip(bands, outs):
        lo, hi = 1 + 128 * b, min(n, 128 * e) + 1
        full[..., :, lo:hi] = o[..., :, lo:hi]
    got = full.cpu().numpy()
    for i in range(batch):
        np.testing.assert_array_equal(got[i], O.nw(sim[i], 10))


def test_nw_more_strips_than_sms_and_large_index():
    """n = 20000: 157 strips on 148 persistent CTAs (a second wave) and
    (n+1)^2 > 2^28 score words, against the C DP."""
    rng = np.random.default_rng(20)
    n = 20000
    sim = rng.integers(-10, 11, size=(n, n), dtype=np.int32)
    got = K.nw_score(torch.from_numpy(sim).cuda(), 10).cpu().numpy()
    np.testing.assert_array_equal(got, O.nw(sim, 10))


def test_remap_sharded_single_rank_uses_the_gpu_map():
    """shard.remap_sharded on one rank (no process group): the GPU map of the
    local range, bucketing and placement reproduce kernels.remap."""
    import paper_2505_08091_b200 as L
    from paper_2505_08091_b200 import shard
    g = L.parse_layout("GroupBy([2048,2048]).OrderBy(GenP([2048,2048], antidiag))")
    x = torch.arange(2048 * 2048, device="cuda", dtype=torch.int32)
    assert torch.equal(shard.remap_sharded(x, g), K.remap(x, None, g))
