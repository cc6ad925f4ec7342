// gemm_tcgen05.cu -- bf16 GEMM on 5th-generation tensor cores (config 5).
//
//   C[b] (M x N, bf16, row-major) = A[b] (M x K, row-major) * B[b]^T (B is N x K row-major)
//
// Blackwell-native structure, written directly in PTX:
//  * persistent kernel, one CTA per SM, 6 warps with fixed roles:
//      warp 0      TMA producer (one elected lane): cp.async.bulk.tensor into a
//                  4-stage smem ring (A 128x64, B 256x64 bf16 per stage, 128-byte
//                  swizzle), completion via mbarrier transaction counts
//      warp 1      TMEM allocator (whole warp) + MMA issuer (one lane):
//                  tcgen05.mma.cta_group::1.kind::f16, M=128 N=256 K=16, fp32
//                  accumulators in TMEM, double-buffered (2 x 256 columns) so the
//                  epilogue of tile i overlaps the main loop of tile i+1;
//                  tcgen05.commit releases smem stages / publishes accumulators
//      warps 2..5  epilogue: tcgen05.ld 32x32b -> bf16 -> global
//  * LEGO-specified CTA raster: the output-tile index walks the layout
//        GroupBy([MB/G, NB, G]).OrderBy(Row(MB/G, NB, G))  (tiles grouped G
//    m-blocks at a time so the ~148 live tiles share A/B panels in L2); the
//    kernel evaluates that layout's inverse (tile_coords below), which
//    tests/test_gemm_raster.py derives with inv_symbolic and checks.
//  * smem operand layouts are the UMMA canonical K-major SWIZZLE_128B atoms
//    (8 rows x 128 B, XOR of 16-byte chunks by row % 8) that TMA produces.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <mutex>

#include "lego_common.h"

namespace {

constexpr int BM = 128, BN = 256, BK = 64;          // CTA tile (K step = one 128-byte swizzle row)
constexpr int STAGES = 4;
constexpr int UMMA_K = 16;
constexpr int A_BYTES = BM * BK * 2;                // 16 KiB
constexpr int B_BYTES = BN * BK * 2;                // 32 KiB
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int NUM_THREADS = 192;
constexpr int ACC_COLS = BN;                        // fp32 accumulator columns per buffer
constexpr int TMEM_COLS = 2 * ACC_COLS;             // double buffered: 512 columns
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;

// ---- PTX wrappers ---------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}"
        :: "r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                            int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5}], [%2];"
        :: "r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1),
           "r"(c2)
        : "memory");
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
    asm volatile("prefetch.tensormap [%0];" :: "l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                 :: "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tc_mma(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                       uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
        :: "r"(d_tmem), "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ bool elect_one() {
    uint32_t pred = 0;
    asm volatile(
        "{\n\t.reg .pred P;\n\t"
        "elect.sync _|P, 0xffffffff;\n\t"
        "selp.b32 %0, 1, 0, P;\n\t}"
        : "=r"(pred));
    return pred != 0;
}

// UMMA shared-memory descriptor: K-major, SWIZZLE_128B, 8-row atoms 1024 B apart
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((addr & 0x3FFFF) >> 4);         // start address        [0,14)
    d |= static_cast<uint64_t>(1) << 16;                        // LBO (unused, 1)      [16,30)
    d |= static_cast<uint64_t>(1024 >> 4) << 32;                // SBO = 1024 B         [32,46)
    d |= static_cast<uint64_t>(1) << 46;                        // version = 1 (sm100)  [46,48)
    d |= static_cast<uint64_t>(2) << 61;                        // SWIZZLE_128B         [61,64)
    return d;
}

// UMMA shared-memory descriptor: MN-major, SWIZZLE_128B.  Canonical layout
// (in 16-byte units) ((8,n),(8,k)):((1,LBO),(8,SBO)): 64 MN-elements x 8 k-rows
// per 1024-byte atom, k-row groups SBO = 1024 B apart, 64-element MN groups
// LBO = 8 KiB apart (one 64 x 64 TMA box per MN group).
__device__ __forceinline__ uint64_t smem_desc_mn(uint32_t addr) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((addr & 0x3FFFF) >> 4);         // start address        [0,14)
    d |= static_cast<uint64_t>(8192 >> 4) << 16;                // LBO = 8 KiB          [16,30)
    d |= static_cast<uint64_t>(1024 >> 4) << 32;                // SBO = 1024 B         [32,46)
    d |= static_cast<uint64_t>(1) << 46;                        // version = 1 (sm100)  [46,48)
    d |= static_cast<uint64_t>(2) << 61;                        // SWIZZLE_128B         [61,64)
    return d;
}

// instruction descriptor: kind::f16, A/B bf16 K-major, D fp32, M=128, N=256
__host__ __device__ constexpr uint32_t make_idesc() {
    return (1u << 4)                       // D format F32
           | (1u << 7)                     // A format BF16
           | (1u << 10)                    // B format BF16
           | (uint32_t(BN >> 3) << 17)     // N >> 3
           | (uint32_t(BM >> 4) << 24);    // M >> 4
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
    uint32_t r;
    asm("cvt.rn.bf16x2.f32 %0, %2, %1;" : "=r"(r) : "f"(lo), "f"(hi));
    return r;
}

// 32 lanes x 32 consecutive fp32 accumulator columns (no wait)
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
          "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
          "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
          "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
}

// LEGO raster: tile t -> (batch, m-block, n-block).  The layout
//   GroupBy([MB/G, NB, G]).OrderBy(Row(MB/G, NB, G)),  inv(t) = (g, n, m_in)
// lists tiles group by group (G m-blocks), n-blocks inside a group,
// m fastest; m-block = g*G + m_in.  Falls back to G = MB % G tail groups.
struct Raster {
    int mb, nb, per_batch, group;                          // group = G (m-blocks per group)
    __device__ __forceinline__ void coords(int t, int& b, int& m, int& n) const {
        b = t / per_batch;
        int r = t - b * per_batch;
        const int G = group;
        const int full = (mb / G) * G;                     // m-blocks in complete groups
        const int g_tiles = G * nb;
        if (r < (full / G) * g_tiles || full == mb) {
            const int g = r / g_tiles;
            const int rem = r - g * g_tiles;
            n = rem / G;
            m = g * G + (rem - n * G);
        } else {                                           // tail group of mb % G m-blocks
            const int tail = mb - full;
            const int rem = r - (full / G) * g_tiles;
            n = rem / tail;
            m = full + (rem - n * tail);
        }
    }
};

// tile t -> (batch, m-block, n-block): the LEGO grouped raster (raster_mode =
// G > 0) or row-major (0).  The only tile-order arithmetic of both GEMM
// kernels; lego_gemm_raster dumps it for tests/test_gemm_raster.py, which
// compares it with the LEGO layout's inverse map on the device.
__device__ __forceinline__ void tile_coords(const Raster& ras, int raster_mode, int t, int& b, int& m, int& n) {
    if (raster_mode) {
        ras.coords(t, b, m, n);
    } else {
        b = t / ras.per_batch;
        const int r = t - b * ras.per_batch;
        m = r / ras.nb;
        n = r - m * ras.nb;
    }
}

__global__ void gemm_raster_dump(int* __restrict__ out, int mtiles, int ntiles, int batch, int raster_mode) {
    const Raster ras{mtiles, ntiles, mtiles * ntiles, raster_mode > 0 ? raster_mode : 1};
    const int total = ras.per_batch * batch;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
        int b, m, n;
        tile_coords(ras, raster_mode, t, b, m, n);
        out[3 * t] = b;
        out[3 * t + 1] = m;
        out[3 * t + 2] = n;
    }
}

__global__ void __launch_bounds__(NUM_THREADS, 1)
gemm_bf16_tcgen05(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_b,
                  __nv_bfloat16* __restrict__ C, int M, int N, int K, int batch, int raster_mode) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    unsigned char* sA = smem;
    unsigned char* sB = smem + STAGES * A_BYTES;
    uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
    uint64_t* empty_bar = full_bar + STAGES;
    uint64_t* acc_full = empty_bar + STAGES;       // [2]
    uint64_t* acc_empty = acc_full + 2;            // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int kblocks = K / BK;
    // raster_mode: 0 = row-major tile order, G > 0 = LEGO grouped raster with G m-blocks per group
    Raster ras{M / BM, N / BN, (M / BM) * (N / BN), raster_mode > 0 ? raster_mode : 1};
    const int total_tiles = ras.per_batch * batch;

    if (warp == 0 && lane == 0) {
        prefetch_tmap(&tmap_a);
        prefetch_tmap(&tmap_b);
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full_bar[s], 1);
            mbar_init(&empty_bar[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&acc_full[a], 1);
            mbar_init(&acc_empty[a], 4);            // one arrive per epilogue warp
        }
        fence_barrier_init();
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                     :: "r"(smem_u32(tmem_slot)), "r"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        // ===================== TMA producer =====================
        if (elect_one()) {
            int stage = 0;
            uint32_t phase = 0;
            for (int t = blockIdx.x; t < total_tiles; t += gridDim.x) {
                int b, mb, nb;
                tile_coords(ras, raster_mode, t, b, mb, nb);
                for (int kb = 0; kb < kblocks; ++kb) {
                    mbar_wait(&empty_bar[stage], phase ^ 1);
                    mbar_expect_tx(&full_bar[stage], STAGE_BYTES);
                    tma_load_3d(sA + stage * A_BYTES, &tmap_a, &full_bar[stage], kb * BK, mb * BM, b);
                    tma_load_3d(sB + stage * B_BYTES, &tmap_b, &full_bar[stage], kb * BK, nb * BN, b);
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        // ===================== MMA issuer =====================
        constexpr uint32_t idesc = make_idesc();
        int stage = 0;
        uint32_t phase = 0;
        int it = 0;
        for (int t = blockIdx.x; t < total_tiles; t += gridDim.x, ++it) {
            const int acc = it & 1;
            const uint32_t acc_phase = (it >> 1) & 1;
            mbar_wait(&acc_empty[acc], acc_phase ^ 1);
            tc_fence_after();
            const uint32_t d_tmem = tmem_base + acc * ACC_COLS;
            for (int kb = 0; kb < kblocks; ++kb) {
                mbar_wait(&full_bar[stage], phase);
                tc_fence_after();
                if (elect_one()) {
                    const uint32_t a0 = smem_u32(sA + stage * A_BYTES);
                    const uint32_t b0 = smem_u32(sB + stage * B_BYTES);
#pragma unroll
                    for (int k = 0; k < BK / UMMA_K; ++k) {
                        // advancing along K inside the 128-byte swizzle row = +32 B per UMMA_K
                        tc_mma(d_tmem, smem_desc(a0 + k * UMMA_K * 2), smem_desc(b0 + k * UMMA_K * 2), idesc,
                               (kb | k) != 0);
                    }
                    tc_commit(&empty_bar[stage]);           // smem slot free once these MMAs finish
                    if (kb == kblocks - 1) tc_commit(&acc_full[acc]);
                }
                __syncwarp();
                if (++stage == STAGES) { stage = 0; phase ^= 1; }
            }
        }
    } else {
        // ===================== epilogue (warps 2..5) =====================
        const int quarter = warp & 3;                         // TMEM lanes 32*quarter .. +31
        int it = 0;
        for (int t = blockIdx.x; t < total_tiles; t += gridDim.x, ++it) {
            int b, mb, nb;
            tile_coords(ras, raster_mode, t, b, mb, nb);
            const int acc = it & 1;
            mbar_wait(&acc_full[acc], (it >> 1) & 1);
            tc_fence_after();
            const int row = mb * BM + quarter * 32 + lane;
            __nv_bfloat16* crow = C + (static_cast<size_t>(b) * M + row) * static_cast<size_t>(N) + nb * BN;
            const uint32_t taddr = tmem_base + acc * ACC_COLS + (static_cast<uint32_t>(quarter * 32) << 16);
#pragma unroll 1
            for (int c = 0; c < BN; c += 32) {
                uint32_t v[32];
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
                    "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                    "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                    : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                      "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
                      "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
                      "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
                      "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                    : "r"(taddr + c));
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                uint4* dst = reinterpret_cast<uint4*>(crow + c);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    uint4 o;
                    o.x = pack_bf16(__uint_as_float(v[8 * q + 0]), __uint_as_float(v[8 * q + 1]));
                    o.y = pack_bf16(__uint_as_float(v[8 * q + 2]), __uint_as_float(v[8 * q + 3]));
                    o.z = pack_bf16(__uint_as_float(v[8 * q + 4]), __uint_as_float(v[8 * q + 5]));
                    o.w = pack_bf16(__uint_as_float(v[8 * q + 6]), __uint_as_float(v[8 * q + 7]));
                    dst[q] = o;
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&acc_empty[acc]);
        }
    }
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem_base), "r"(TMEM_COLS));
    }
}

// ===========================================================================
// CTA-pair variant (cta_group::2): a cluster of 2 CTAs on one TPC computes a
// 256 x 256 output tile with tcgen05.mma.cta_group::2 (M = 256): each CTA
// stages its own 128 rows of A and its own 128-row half of B (so every
// operand byte crosses L2 -> SM once per pair instead of twice), the leader
// CTA's single thread issues the MMAs for both, and each CTA's TMEM holds its
// 128 accumulator rows.  Barrier protocol:
//   full[s]     leader only; the leader arrives with expect_tx(both CTAs'
//               bytes) and both CTAs' TMA loads complete_tx on it
//   empty[s]    both CTAs; the leader's tcgen05.commit multicasts to both
//   acc_full[a] both CTAs; multicast commit after a tile's last k-block
//   acc_empty[a] leader only; the 4 epilogue warps of each CTA arrive (8)
namespace pair {

// NH = number of N=256 halves per pair tile: 1 -> 256 x 256 tiles with a
// double-buffered accumulator (epilogue overlaps the next tile), 2 -> 256 x 512
// tiles (each operand byte feeds 4/3 more FLOPs; the 512-column accumulator
// fills TMEM, so the epilogue of a tile precedes the next tile's MMAs)
template <int NH>
struct Cfg {
    static constexpr int BM = 128;                   // rows of A per CTA (pair M = 256)
    static constexpr int BN = 256 * NH;              // pair N
    static constexpr int BNH = 128 * NH;             // rows of B staged per CTA
    static constexpr int BK = 64;
    static constexpr int STAGES = NH == 1 ? 6 : 4;
    static constexpr int A_BYTES = BM * BK * 2;      // 16 KiB
    static constexpr int B_BYTES = BNH * BK * 2;     // 16 KiB per half
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    // warps: 0 TMA, 1 MMA, then 4 epilogue warps per 256 accumulator columns
    static constexpr int NUM_THREADS = 64 + 128 * NH;
    static constexpr int ACC_COLS = BN;
    static constexpr int NBUF = NH == 1 ? 2 : 1;     // accumulator buffers in TMEM
    static constexpr int TMEM_COLS = 512;
    static constexpr int EPI_BYTES = 2048;           // per epilogue warp: 32 rows x 64 B staging
    static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 + 256 + (NUM_THREADS / 32 - 2) * EPI_BYTES;
};
constexpr int BM = 128, BN = 256;                    // host-side geometry checks (NH = 1 tile)

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t map_to_cta(uint32_t addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" :: "r"(cluster_addr) : "memory");
}
// TMA into this CTA's smem, completion signalled on an mbarrier of either CTA of the pair
__device__ __forceinline__ void tma_load_3d_pair(void* dst, const CUtensorMap* map, uint32_t bar_cluster, int c0,
                                                 int c1, int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5}], [%2];"
        :: "r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(bar_cluster), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}
__device__ __forceinline__ void tc_mma2(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                        uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}"
        :: "r"(d_tmem), "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void tc_commit2(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                 :: "r"(smem_u32(bar)), "h"((uint16_t)0x3) : "memory");
}

// M = 256 (cta_group::2), N = 256 per instruction
__host__ __device__ constexpr uint32_t make_idesc2() {
    return (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(256 >> 3) << 17) | (uint32_t(256 >> 4) << 24);
}

// operand majors: TA / TB = the operand is stored MN-major ("Col" data layout:
// A as K x M, B as K x N row-major), else K-major (A as M x K, B as N x K)
template <int NH, bool TA, bool TB>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(Cfg<NH>::NUM_THREADS, 1)
gemm_bf16_tcgen05_pair(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_b,
                       __nv_bfloat16* __restrict__ C, int M, int N, int K, int batch, int raster_mode) {
    using C_ = Cfg<NH>;
    constexpr int BM = C_::BM, BN = C_::BN, BK = C_::BK, STAGES = C_::STAGES;
    constexpr int A_BYTES = C_::A_BYTES, B_BYTES = C_::B_BYTES, STAGE_BYTES = C_::STAGE_BYTES;
    constexpr int ACC_COLS = C_::ACC_COLS, NBUF = C_::NBUF, TMEM_COLS = C_::TMEM_COLS;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    unsigned char* sA = smem;
    unsigned char* sB = smem + STAGES * A_BYTES;
    uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
    uint64_t* empty_bar = full_bar + STAGES;
    uint64_t* acc_full = empty_bar + STAGES;       // [NBUF]
    uint64_t* acc_empty = acc_full + 2;            // [NBUF]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
    unsigned char* epi_stage = smem + STAGES * STAGE_BYTES + 256;      // [epilogue warp][32 rows][64 B]

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t rank = cluster_rank();
    const bool leader = rank == 0;
    // ragged shapes: the last k-block / tile rows / tile columns run past K, M, N;
    // TMA zero-fills the operand boxes there and the epilogue masks the stores
    const int kblocks = (K + BK - 1) / BK;
    const int mtiles = (M + 2 * BM - 1) / (2 * BM), ntiles = (N + BN - 1) / BN;
    // tiles are 256-row "m-blocks" x BN columns
    Raster ras{mtiles, ntiles, mtiles * ntiles, raster_mode > 0 ? raster_mode : 1};
    const int total_tiles = ras.per_batch * batch;
    const int pair_id = blockIdx.x >> 1, num_pairs = gridDim.x >> 1;

    if (warp == 0 && lane == 0) {
        prefetch_tmap(&tmap_a);
        prefetch_tmap(&tmap_b);
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full_bar[s], 1);
            mbar_init(&empty_bar[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&acc_full[a], 1);
            mbar_init(&acc_empty[a], 8);            // 4 epilogue warps x 2 CTAs
        }
        fence_barrier_init();
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;"
                     :: "r"(smem_u32(tmem_slot)), "r"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    // the leader's barriers, as shared::cluster addresses
    const uint32_t full_leader = map_to_cta(smem_u32(full_bar), 0);
    const uint32_t acc_empty_leader = map_to_cta(smem_u32(acc_empty), 0);

    auto coords = [&](int t, int& b, int& m, int& n) { tile_coords(ras, raster_mode, t, b, m, n); };

    if (warp == 0) {
        // ===================== TMA producer (both CTAs) =====================
        if (elect_one()) {
            int stage = 0;
            uint32_t phase = 0;
            for (int t = pair_id; t < total_tiles; t += num_pairs) {
                int b, mb, nb;
                coords(t, b, mb, nb);
                const int arow = mb * 2 * BM + (int)rank * BM;
                for (int kb = 0; kb < kblocks; ++kb) {
                    mbar_wait(&empty_bar[stage], phase ^ 1);
                    if (leader) mbar_expect_tx(&full_bar[stage], 2 * STAGE_BYTES);
                    const uint32_t fb = full_leader + 8u * stage;
                    if (TA) {                                   // two 64(M) x 64(K) boxes
                        tma_load_3d_pair(sA + stage * A_BYTES, &tmap_a, fb, arow, kb * BK, b);
                        tma_load_3d_pair(sA + stage * A_BYTES + 8192, &tmap_a, fb, arow + 64, kb * BK, b);
                    } else {
                        tma_load_3d_pair(sA + stage * A_BYTES, &tmap_a, fb, kb * BK, arow, b);
                    }
                    // B half h: this CTA's 128 rows of the output columns [256h, 256h + 256)
#pragma unroll
                    for (int h = 0; h < NH; ++h) {
                        const int brow = nb * BN + h * 256 + (int)rank * 128;
                        unsigned char* dstb = sB + stage * B_BYTES + h * (128 * BK * 2);
                        if (TB) {
                            tma_load_3d_pair(dstb, &tmap_b, fb, brow, kb * BK, b);
                            tma_load_3d_pair(dstb + 8192, &tmap_b, fb, brow + 64, kb * BK, b);
                        } else {
                            tma_load_3d_pair(dstb, &tmap_b, fb, kb * BK, brow, b);
                        }
                    }
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        // ===================== MMA issuer (leader CTA only) =====================
        if (leader) {
            constexpr uint32_t idesc = make_idesc2() | (uint32_t(TA) << 15) | (uint32_t(TB) << 16);
            // K step k (16 elements): +32 B inside the K-major swizzle row, or +2 atoms (2 x 8 k-rows)
            auto adesc = [](uint32_t base, int k) {
                return TA ? smem_desc_mn(base + k * 2048) : smem_desc(base + k * UMMA_K * 2);
            };
            auto bdesc = [](uint32_t base, int k) {
                return TB ? smem_desc_mn(base + k * 2048) : smem_desc(base + k * UMMA_K * 2);
            };
            int stage = 0;
            uint32_t phase = 0;
            int it = 0;
            for (int t = pair_id; t < total_tiles; t += num_pairs, ++it) {
                const int acc = NBUF == 2 ? (it & 1) : 0;
                const uint32_t acc_phase = NBUF == 2 ? ((it >> 1) & 1) : (it & 1);
                // NH == 2: acc_empty[h] = accumulator columns [256h, 256h+256) drained
                mbar_wait(&acc_empty[acc], acc_phase ^ 1);
                tc_fence_after();
                const uint32_t d_tmem = tmem_base + acc * ACC_COLS;
                for (int kb = 0; kb < kblocks; ++kb) {
                    mbar_wait(&full_bar[stage], phase);
                    tc_fence_after();
                    if (NH == 2 && kb == 0) {
                        // first k-block: half 0 while the epilogue still drains half 1
                        const uint32_t a0 = smem_u32(sA + stage * A_BYTES);
                        const uint32_t b0 = smem_u32(sB + stage * B_BYTES);
                        if (elect_one()) {
#pragma unroll
                            for (int k = 0; k < BK / UMMA_K; ++k)
                                tc_mma2(d_tmem, adesc(a0, k), bdesc(b0, k), idesc, k != 0);
                        }
                        __syncwarp();
                        mbar_wait(&acc_empty[1], acc_phase ^ 1);
                        tc_fence_after();
                        if (elect_one()) {
#pragma unroll
                            for (int k = 0; k < BK / UMMA_K; ++k)
                                tc_mma2(d_tmem + 256, adesc(a0, k), bdesc(b0 + 128 * BK * 2, k), idesc, k != 0);
                            tc_commit2(&empty_bar[stage]);
                            if (kb == kblocks - 1) tc_commit2(&acc_full[acc]);
                        }
                        __syncwarp();
                        if (++stage == STAGES) { stage = 0; phase ^= 1; }
                        continue;
                    }
                    if (elect_one()) {
                        const uint32_t a0 = smem_u32(sA + stage * A_BYTES);
                        const uint32_t b0 = smem_u32(sB + stage * B_BYTES);
#pragma unroll
                        for (int k = 0; k < BK / UMMA_K; ++k)
#pragma unroll
                            for (int h = 0; h < NH; ++h)
                                tc_mma2(d_tmem + h * 256, adesc(a0, k), bdesc(b0 + h * (128 * BK * 2), k), idesc,
                                        (kb | k) != 0);
                        tc_commit2(&empty_bar[stage]);
                        if (kb == kblocks - 1) tc_commit2(&acc_full[acc]);
                    }
                    __syncwarp();
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else {
        // ===================== epilogue (warps 2.., both CTAs) =====================
        // warp -> TMEM lane quarter (warp % 4) and accumulator half (NH == 2)
        const int quarter = warp & 3;
        const int half = (warp - 2) >> 2;
        constexpr int EPI_COLS = 256;                         // columns per epilogue warp
#ifndef LEGO_GEMM_EPI_CHUNKS
#define LEGO_GEMM_EPI_CHUNKS 4                              // measured: 4 chunks 681 us, 2 chunks 689 us (8192^3)
#endif
        constexpr int EPI_CHUNKS = LEGO_GEMM_EPI_CHUNKS;      // 32-column TMEM loads in flight
        int it = 0;
        for (int t = pair_id; t < total_tiles; t += num_pairs, ++it) {
            int b, mb, nb;
            coords(t, b, mb, nb);
            const int acc = NBUF == 2 ? (it & 1) : 0;
            mbar_wait(&acc_full[acc], NBUF == 2 ? ((it >> 1) & 1) : (it & 1));
            tc_fence_after();
            const int row0 = mb * 2 * BM + (int)rank * BM + quarter * 32;      // this warp's 32 rows
            __nv_bfloat16* cbase = C + (static_cast<size_t>(b) * M + row0) * static_cast<size_t>(N) + nb * BN +
                                   half * EPI_COLS;
            // staging: row r's 16-byte chunk q at r*64 + 16*(q ^ ((r >> 1) & 3)) -- conflict-free for
            // both the row-per-lane writes and the 4-lanes-per-row reads
            unsigned char* stg = epi_stage + (warp - 2) * C_::EPI_BYTES;
            const uint32_t taddr = tmem_base + acc * ACC_COLS + half * EPI_COLS +
                                   (static_cast<uint32_t>(quarter * 32) << 16);
#ifndef LEGO_GEMM_EARLY_RELEASE
#define LEGO_GEMM_EARLY_RELEASE 1
#endif
#if LEGO_GEMM_EARLY_RELEASE
            // drain the whole half into registers as packed bf16 pairs (128 words),
            // release the TMEM columns to the MMA warp, then stage and store: the
            // next tile's MMAs into this half overlap this tile's global stores
            {
                uint32_t pk[EPI_COLS / 2];
#pragma unroll
                for (int c = 0; c < EPI_COLS; c += 32 * EPI_CHUNKS) {
                    uint32_t v[EPI_CHUNKS][32];
#pragma unroll
                    for (int h2 = 0; h2 < EPI_CHUNKS; ++h2) tmem_ld32(taddr + c + 32 * h2, v[h2]);
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                    for (int h2 = 0; h2 < EPI_CHUNKS; ++h2)
#pragma unroll
                        for (int j = 0; j < 16; ++j)
                            pk[(c + 32 * h2) / 2 + j] = pack_bf16(__uint_as_float(v[h2][2 * j]),
                                                                  __uint_as_float(v[h2][2 * j + 1]));
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive_cluster(acc_empty_leader + 8u * (NH == 2 ? half : acc));
#pragma unroll
                for (int c = 0; c < EPI_COLS; c += 32) {
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const uint4 o = make_uint4(pk[c / 2 + 4 * q + 0], pk[c / 2 + 4 * q + 1],
                                                   pk[c / 2 + 4 * q + 2], pk[c / 2 + 4 * q + 3]);
                        *reinterpret_cast<uint4*>(stg + lane * 64 + 16 * (q ^ ((lane >> 1) & 3))) = o;
                    }
                    __syncwarp();
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int r = 8 * q + (lane >> 2), cq = lane & 3;
                        const uint4 o = *reinterpret_cast<const uint4*>(stg + r * 64 + 16 * (cq ^ ((r >> 1) & 3)));
                        const int gcol = nb * BN + half * EPI_COLS + c + 8 * cq;     // N % 8 == 0
                        if (row0 + r < M && gcol < N)
                            *reinterpret_cast<uint4*>(cbase + static_cast<size_t>(r) * N + c + 8 * cq) = o;
                    }
                    __syncwarp();
                }
            }
#else
#pragma unroll 1
#ifdef LEGO_GEMM_ABL_NOEPI
            if (M < 0)                                          // ablation: skip the epilogue body
#endif
            for (int c = 0; c < EPI_COLS; c += 32 * EPI_CHUNKS) {
                uint32_t v[EPI_CHUNKS][32];                     // EPI_CHUNKS x 32 columns per TMEM round trip
#pragma unroll
                for (int h2 = 0; h2 < EPI_CHUNKS; ++h2) tmem_ld32(taddr + c + 32 * h2, v[h2]);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                for (int h2 = 0; h2 < EPI_CHUNKS; ++h2) {
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        uint4 o;
                        o.x = pack_bf16(__uint_as_float(v[h2][8 * q + 0]), __uint_as_float(v[h2][8 * q + 1]));
                        o.y = pack_bf16(__uint_as_float(v[h2][8 * q + 2]), __uint_as_float(v[h2][8 * q + 3]));
                        o.z = pack_bf16(__uint_as_float(v[h2][8 * q + 4]), __uint_as_float(v[h2][8 * q + 5]));
                        o.w = pack_bf16(__uint_as_float(v[h2][8 * q + 6]), __uint_as_float(v[h2][8 * q + 7]));
                        *reinterpret_cast<uint4*>(stg + lane * 64 + 16 * (q ^ ((lane >> 1) & 3))) = o;
                    }
                    __syncwarp();
                    // 4 lanes per row: each store instruction writes 8 full 64-byte row segments
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int r = 8 * q + (lane >> 2), cq = lane & 3;
                        const uint4 o = *reinterpret_cast<const uint4*>(stg + r * 64 + 16 * (cq ^ ((r >> 1) & 3)));
                        const int gcol = nb * BN + half * EPI_COLS + c + 32 * h2 + 8 * cq;   // N % 8 == 0
                        if (row0 + r < M && gcol < N)
                            *reinterpret_cast<uint4*>(cbase + static_cast<size_t>(r) * N + c + 32 * h2 + 8 * cq) = o;
                    }
                    __syncwarp();
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(acc_empty_leader + 8u * (NH == 2 ? half : acc));
#endif
        }
    }
    tc_fence_before();
    cluster_sync();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" :: "r"(tmem_base), "r"(TMEM_COLS));
    }
}

}  // namespace pair

// ---- host side ------------------------------------------------------------
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    });
    return fn;
}

// MN-major operand stored K x rows row-major (rows contiguous): box = 64 rows x 64 k
lego_status make_map_mn(CUtensorMap* map, const void* base, int64_t rows, int64_t K, int64_t batch) {
    EncodeTiledFn enc = encode_fn();
    if (!enc) return lego_fail(LEGO_E_CUDA, "cuTensorMapEncodeTiled unavailable");
    cuuint64_t dims[3] = {(cuuint64_t)rows, (cuuint64_t)K, (cuuint64_t)batch};
    cuuint64_t strides[2] = {(cuuint64_t)rows * 2, (cuuint64_t)(rows * K * 2)};
    cuuint32_t box[3] = {64, BK, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return lego_fail(LEGO_E_CUDA, "cuTensorMapEncodeTiled (MN-major) failed (%d)", (int)r);
    return LEGO_OK;
}

lego_status make_map(CUtensorMap* map, const void* base, int64_t rows, int64_t K, int64_t batch, int box_rows) {
    EncodeTiledFn enc = encode_fn();
    if (!enc) return lego_fail(LEGO_E_CUDA, "cuTensorMapEncodeTiled unavailable");
    cuuint64_t dims[3] = {(cuuint64_t)K, (cuuint64_t)rows, (cuuint64_t)batch};
    cuuint64_t strides[2] = {(cuuint64_t)K * 2, (cuuint64_t)(rows * K * 2)};
    cuuint32_t box[3] = {BK, (cuuint32_t)box_rows, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return lego_fail(LEGO_E_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    return LEGO_OK;
}

template <int NH, bool TA, bool TB>
lego_status launch_pair(const CUtensorMap& ma, const CUtensorMap& mb, void* C, int64_t M, int64_t N, int64_t K,
                        int64_t batch, int raster, int64_t pairs, void* stream) {
    using C_ = pair::Cfg<NH>;
    static std::atomic<unsigned long long> attr_set{0};
    LEGO_TRY(lego_smem_optin(pair::gemm_bf16_tcgen05_pair<NH, TA, TB>, C_::SMEM_BYTES, attr_set,
                             "cudaFuncSetAttribute(gemm pair smem)"));
    pair::gemm_bf16_tcgen05_pair<NH, TA, TB><<<(unsigned)(2 * pairs), C_::NUM_THREADS, C_::SMEM_BYTES,
                                               static_cast<cudaStream_t>(stream)>>>(
        ma, mb, static_cast<__nv_bfloat16*>(C), (int)M, (int)N, (int)K, (int)batch, raster);
    return lego_cuda_check(cudaGetLastError(), "gemm pair launch");
}

bool pair_wide() {
    static const bool w = [] {
        const char* e = getenv("LEGO_GEMM_WIDE");
        return !(e && e[0] == '0');
    }();
    return w;
}

template <int NH>
lego_status dispatch_pair(bool ta, bool tb, const CUtensorMap& ma, const CUtensorMap& mb, void* C, int64_t M,
                          int64_t N, int64_t K, int64_t batch, int raster, int64_t pairs, void* stream) {
    if (ta && tb) return launch_pair<NH, true, true>(ma, mb, C, M, N, K, batch, raster, pairs, stream);
    if (ta) return launch_pair<NH, true, false>(ma, mb, C, M, N, K, batch, raster, pairs, stream);
    if (tb) return launch_pair<NH, false, true>(ma, mb, C, M, N, K, batch, raster, pairs, stream);
    return launch_pair<NH, false, false>(ma, mb, C, M, N, K, batch, raster, pairs, stream);
}

lego_status gemm_impl(const void* A, const void* B, void* C, int64_t M, int64_t N, int64_t K, int64_t batch,
                      int32_t raster, int32_t a_major, int32_t b_major, void* stream) {
    if (M <= 0 || N <= 0 || K <= 0 || batch <= 0)
        return lego_fail(LEGO_E_SHAPE, "gemm shape must be positive");
    if (a_major < 0 || a_major > 1 || b_major < 0 || b_major > 1)
        return lego_fail(LEGO_E_ARG, "operand major must be 0 (K-major) or 1 (MN-major)");
    const bool ta = a_major == 1, tb = b_major == 1;
    // 16-byte rows for every TMA-read operand and for C
    if (N % 8 || (!ta || !tb ? K % 8 : 0) || (ta && M % 8))
        return lego_fail(LEGO_E_SHAPE,
                         "gemm needs N %% 8 == 0, K %% 8 == 0 (K-major operands), M %% 8 == 0 (MN-major A); "
                         "got M=%lld N=%lld K=%lld", (long long)M, (long long)N, (long long)K);
    if (M * batch > INT32_MAX || N > INT32_MAX || K > INT32_MAX)
        return lego_fail(LEGO_E_SHAPE, "gemm dimensions too large");
    if (((uintptr_t)A | (uintptr_t)B | (uintptr_t)C) & 15)
        return lego_fail(LEGO_E_ARG, "gemm buffers must be 16-byte aligned");
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    static const bool pair_ok = [] {
        const char* e = getenv("LEGO_GEMM_PAIR");
        return !(e && e[0] == '0');
    }();
    // exact tiles: single-CTA 128 x 256 when M % 256 != 0; ragged shapes and MN-major
    // operands go to the pair kernel
    const bool ragged = M % BM || N % BN || K % BK || ta || tb;
    if (ragged || (pair_ok && M % (2 * pair::BM) == 0 && N % pair::BN == 0)) {
        // CTA-pair kernel on cta_group::2: 256 x 512 tiles when N allows, else 256 x 256
        const bool wide = (ragged ? N > 256 : N % 512 == 0) && pair_wide();
        CUtensorMap ma, mb;
        if (ta) LEGO_TRY(make_map_mn(&ma, A, M, K, batch));
        else LEGO_TRY(make_map(&ma, A, M, K, batch, pair::BM));
        if (tb) LEGO_TRY(make_map_mn(&mb, B, N, K, batch));
        else LEGO_TRY(make_map(&mb, B, N, K, batch, 128));
        const int64_t tn = wide ? 512 : 256;
        const int64_t tiles = ((M + 255) / 256) * ((N + tn - 1) / tn) * batch;
        const int64_t pairs = tiles < sms / 2 ? tiles : sms / 2;
        const int g = raster > 1 ? raster / 2 : raster;   // G counts 128-row m-blocks; pair tiles are 256 rows
        if (wide) return dispatch_pair<2>(ta, tb, ma, mb, C, M, N, K, batch, g, pairs, stream);
        return dispatch_pair<1>(ta, tb, ma, mb, C, M, N, K, batch, g, pairs, stream);
    }
    CUtensorMap ma, mb;
    LEGO_TRY(make_map(&ma, A, M, K, batch, BM));
    LEGO_TRY(make_map(&mb, B, N, K, batch, BN));
    static std::atomic<unsigned long long> attr_set{0};
    LEGO_TRY(lego_smem_optin(gemm_bf16_tcgen05, SMEM_BYTES, attr_set, "cudaFuncSetAttribute(gemm smem)"));
    const int64_t tiles = (M / BM) * (N / BN) * batch;
    const int grid = (int)(tiles < sms ? tiles : sms);
    gemm_bf16_tcgen05<<<grid, NUM_THREADS, SMEM_BYTES, static_cast<cudaStream_t>(stream)>>>(
        ma, mb, static_cast<__nv_bfloat16*>(C), (int)M, (int)N, (int)K, (int)batch, raster);
    return lego_cuda_check(cudaGetLastError(), "gemm launch");
}

}  // namespace

extern "C" lego_status lego_gemm_raster(int32_t* out, int64_t mtiles, int64_t ntiles, int64_t batch,
                                        int32_t raster, void* stream) {
    if (mtiles <= 0 || ntiles <= 0 || batch <= 0 || mtiles * ntiles * batch > INT32_MAX / 3)
        return lego_fail(LEGO_E_SHAPE, "bad raster size");
    if (raster < 0) return lego_fail(LEGO_E_ARG, "raster group must be >= 0");
    if (!out) return lego_fail(LEGO_E_ARG, "null buffer");
    const long long total = mtiles * ntiles * batch;
    const unsigned grid = (unsigned)((total + 255) / 256 < 1024 ? (total + 255) / 256 : 1024);
    gemm_raster_dump<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(out, (int)mtiles, (int)ntiles,
                                                                           (int)batch, raster);
    return lego_cuda_check(cudaGetLastError(), "raster dump");
}

extern "C" lego_status lego_gemm_bf16(const void* A, const void* B, void* C, int64_t M, int64_t N, int64_t K,
                                      int64_t batch, int32_t raster, void* stream) {
    return gemm_impl(A, B, C, M, N, K, batch, raster, 0, 0, stream);
}

extern "C" lego_status lego_gemm_bf16_ex(const void* A, const void* B, void* C, int64_t M, int64_t N, int64_t K,
                                         int64_t batch, int32_t raster, int32_t a_major, int32_t b_major,
                                         void* stream) {
    return gemm_impl(A, B, C, M, N, K, batch, raster, a_major, b_major, stream);
}
