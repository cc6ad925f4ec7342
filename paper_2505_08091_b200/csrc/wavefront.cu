// wavefront.cu -- Needleman-Wunsch score matrix as an anti-diagonal wavefront
// (BASELINE.json config 4b).
//
//   S[0][j] = -j*p,  S[i][0] = -i*p,
//   S[i][j] = max(S[i-1][j-1] + sim[i-1][j-1], S[i-1][j] - p, S[i][j-1] - p)
//
// Decomposition (no host loop over diagonals, no grid sync):
//  * the n columns are cut into 128-wide strips, one warp per strip, claimed
//    in order from an atomic ticket, so a strip's left neighbour is always
//    already running;
//  * inside a strip the warp sweeps anti-diagonally over 2x4 cell blocks:
//    lane j owns columns 4j..4j+3 and at step s computes rows 2(s-j) and
//    2(s-j)+1, i.e. every step is one anti-diagonal of the (row pairs x 32
//    lane-columns) grid -- the LEGO antidiag order of the paper's NW kernel
//    (PAPER.md:1298-1301).  The two left values arrive by warp shuffle, the
//    up and diagonal values are the lane's own previous rows: the per-step
//    critical path is one shuffle plus a 5-cell max/add chain for 8 cells,
//    and the step body is branch-free (steps are grouped 16 at a time so all
//    bookkeeping happens once per 32-row block);
//  * sim is staged 32 rows x 128 columns at a time by cp.async one block
//    ahead into a 4-block ring, read back one step early along the
//    anti-diagonal (16-byte, conflict-free); results go to a 2-block ring and
//    leave as coalesced row segments once a block is complete; the strip's
//    last column is then published as tagged 64-bit words (value | launch
//    epoch | row) that the right neighbour's lanes poll directly: one L2
//    round trip per 32 rows both synchronises and delivers the data, with no
//    flags and no fences.
#include <cuda_runtime.h>

#include <cstdint>

#include "lego_common.h"

namespace {

constexpr int TILE = 32;                 // rows per block
constexpr int CPL = 4;                   // columns per lane
constexpr int STRIP = 32 * CPL;          // columns per warp strip
constexpr int SIM_ROWS = 4 * TILE;       // sim ring: 4 blocks
constexpr int OUT_ROWS = 4 * TILE;       // out ring: 4 blocks (flushed three blocks late)
constexpr int RPS = 2;                   // rows per lane per step
constexpr int BND_RING = 2 * TILE;
constexpr int SMEM_BYTES = (SIM_ROWS + OUT_ROWS) * STRIP * 4 + BND_RING * 4;

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async4(uint32_t dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" :: "r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

__device__ __forceinline__ int4 lds128v(uint32_t a) {
    int4 v;
    asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
    return v;
}
__device__ __forceinline__ int lds32v(uint32_t a) {
    int v;
    asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}

__global__ void nw_borders(int32_t* __restrict__ score, long long n, int p, long long batch) {
    const long long w = n + 1;
    const long long total = batch * w;
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < total;
         k += (long long)gridDim.x * blockDim.x) {
        const long long b = k / w, x = k - b * w;
        int32_t* s = score + b * w * w;
        s[x] = (int32_t)(-x * p);          // row 0
        s[x * w] = (int32_t)(-x * p);      // column 0
    }
}

struct Strip {
    const int32_t* simb;
    int32_t* sc;
    int2* my_bnd2;                           // (value, tag) boundary words of this strip
    const int2* left_bnd2;                   // ... and of the strip to the left
    unsigned tag;                            // launch epoch << 21 (rows are < 2^20)
    int n, p, w, col0, lane;
    bool vec_ok;
    uint32_t sim_base, out_base, bnd_base;   // shared-window addresses
    int32_t* out_gen;                        // generic pointer of the out ring
};

// stage sim rows [32k, 32k+32) into ring block k % 4 (one cp.async group)
__device__ __forceinline__ void stage_sim(const Strip& st, int k) {
    // pointer-walking, fully unrolled: ~3 instructions per row (the issue cost
    // of this loop competes with the wavefront steps of the same warp)
    const int rows = min(TILE, st.n - k * TILE);
    uint32_t dst = st.sim_base + (uint32_t)((k & 3) * TILE * STRIP) * 4u;
    if (st.vec_ok) {
        const int32_t* src = st.simb + (long long)k * TILE * st.n + st.col0 + CPL * st.lane;
        const bool ok = st.col0 + CPL * st.lane < st.n;
        dst += 16u * st.lane;
#pragma unroll
        for (int r = 0; r < TILE; ++r) {
            if (ok && r < rows) cp_async16(dst, src);
            dst += STRIP * 4u;
            src += st.n;
        }
    } else {
        const int32_t* src = st.simb + (long long)k * TILE * st.n + st.col0 + st.lane;
        dst += 4u * st.lane;
        for (int r = 0; r < rows; ++r) {
#pragma unroll
            for (int q = 0; q < CPL; ++q)
                if (st.col0 + q * 32 + st.lane < st.n) cp_async4(dst + 128u * q, src + 32 * q);
            dst += STRIP * 4u;
            src += st.n;
        }
    }
    cp_async_commit();
}

// block k enters: sim block k landed, block k+1 in flight
__device__ __forceinline__ void enter_block(const Strip& st, int k, int nblocks) {
    if (k + 1 < nblocks) {
        stage_sim(st, k + 1);
        cp_async_wait_1();
    } else {
        cp_async_wait_all();
    }
    __syncwarp();
}

// Left-boundary batches of BATCH rows.  Lanes 0..BATCH-1 load their row's
// tagged word early (bnd_issue) and check it one batch later (bnd_commit),
// spinning only if the left strip has not published it yet; the value then
// goes to the shared ring that lane 0 reads.  Value and tag arrive in one
// naturally aligned 64-bit store, so one L2 round trip both synchronises and
// delivers the data.
constexpr int BATCH = 8;

__device__ __forceinline__ unsigned long long ld_tagged(const int2* p) {
    unsigned long long w;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(w) : "l"(p) : "memory");
    return w;
}

__device__ __forceinline__ unsigned long long bnd_issue(const Strip& st, int batch) {
    const int row = batch * BATCH + st.lane;
    if (st.w == 0 || st.lane >= BATCH || row >= st.n) return 0;
    return ld_tagged(st.left_bnd2 + row);
}

__device__ __forceinline__ void bnd_commit(const Strip& st, int batch, unsigned long long w) {
    const int row = batch * BATCH + st.lane;
    if (st.lane < BATCH) {
        int v = 0;
        if (st.w == 0) {
            v = -(row + 1) * st.p;               // S[row+1][0]
        } else if (row < st.n) {
            const unsigned want = st.tag | (unsigned)(row + 1);
            while ((unsigned)(w >> 32) != want) w = ld_tagged(st.left_bnd2 + row);
            v = (int)(unsigned)w;
        }
        asm volatile("st.shared.b32 [%0], %1;" :: "r"(st.bnd_base + 4u * (row & (BND_RING - 1))), "r"(v)
                     : "memory");
    }
    __syncwarp();
}

// block k is complete: write its rows out as coalesced row segments
__device__ __forceinline__ void flush_block(const Strip& st, int k) {
    __syncwarp();
    const int32_t* src = st.out_gen + ((k * TILE) & (OUT_ROWS - 1)) * STRIP;
    const long long ld = (long long)st.n + 1;
    const int rows = min(TILE, st.n - k * TILE);
    int32_t* dst = st.sc + (long long)(k * TILE + 1) * ld + st.col0 + 1 + st.lane;
    const int32_t* s = src + st.lane;
    bool ok[CPL];
#pragma unroll
    for (int q = 0; q < CPL; ++q) ok[q] = st.col0 + q * 32 + st.lane < st.n;
#pragma unroll 8
    for (int r = 0; r < rows; ++r) {
#pragma unroll
        for (int q = 0; q < CPL; ++q)
            if (ok[q]) dst[32 * q] = s[32 * q];
        dst += ld;
        s += STRIP;
    }
    __syncwarp();
}

__global__ void __launch_bounds__(32)
nw_strips(const int32_t* __restrict__ sim, int32_t* __restrict__ score, int n, int p, int strips_per_matrix,
          int total_strips, int* __restrict__ ticket, int2* __restrict__ bnd2, unsigned epoch) {
    extern __shared__ __align__(16) int32_t smem[];
    const int lane = threadIdx.x;
    const int n_pad = (n + TILE - 1) / TILE * TILE;
    const int nblocks = n_pad / TILE;
    Strip st;
    st.n = n;
    st.p = p;
    st.lane = lane;
    st.tag = (epoch & 0x7FFu) << 21;
    st.vec_ok = (n % 4) == 0;
    st.sim_base = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
    st.out_base = st.sim_base + SIM_ROWS * STRIP * 4;
    st.bnd_base = st.out_base + OUT_ROWS * STRIP * 4;
    st.out_gen = smem + SIM_ROWS * STRIP;

    for (;;) {
        int strip = 0;
        if (lane == 0) strip = atomicAdd(ticket, 1);
        strip = __shfl_sync(0xffffffffu, strip, 0);
        if (strip >= total_strips) return;
        const int b = strip / strips_per_matrix;
        st.w = strip - b * strips_per_matrix;
        st.simb = sim + (long long)b * n * n;
        st.sc = score + (long long)b * ((long long)n + 1) * ((long long)n + 1);
        st.my_bnd2 = bnd2 + (long long)strip * n_pad;
        st.left_bnd2 = st.my_bnd2 - n_pad;
        st.col0 = st.w * STRIP;
        const int c_lane = st.col0 + CPL * lane;

        stage_sim(st, 0);
        // h: the lane's 4 cells of the last finished row (S[0][c+1..c+4] to start);
        // t3: the last cell of the row before it (sent to the right with h3)
        int32_t h0 = -(c_lane + 1) * p, h1 = -(c_lane + 2) * p, h2 = -(c_lane + 3) * p,
                h3 = -(c_lane + 4) * p, t3 = 0;
        int32_t left_prev = -c_lane * p;                    // S[i][c_lane] of the last finished row i

        // boundary batches: 0 committed now, 1 in flight (committed at step 0)
        bnd_commit(st, 0, bnd_issue(st, 0));
        unsigned long long bnd_pending = bnd_issue(st, 1);
        const int nbatches = (n + BATCH - 1) / BATCH;

        // a block of 32 rows is 16 steps for lane 0 (two rows per step); lane 31 runs
        // 31 steps behind, so block k completes at step 16k + 46 and is flushed at
        // the start of block k + 3
        for (int k = 0; k <= nblocks + 2; ++k) {
            if (k >= 3) flush_block(st, k - 3);
            if (k > nblocks + 1) break;
            if (k < nblocks) enter_block(st, k, nblocks);
            int4* out_ring = reinterpret_cast<int4*>(st.out_gen) + lane;
            const uint32_t sim_lane = st.sim_base + 16u * lane;   // + row * STRIP*4
            // sim rows run PF steps ahead in a register queue (static indices under full
            // unrolling); refilled at every block start because lane 0's prefetches past
            // the block edge may have read unlanded rows
            constexpr int PF = 2;
            int4 sq0[PF], sq1[PF];
            int bq0[PF], bq1[PF];
#pragma unroll
            for (int d = 0; d < PF; ++d) {
                const int s = k * (TILE / RPS) + d;
                const int r = RPS * (s - lane);
                sq0[d] = lds128v(sim_lane + (uint32_t)((r & (SIM_ROWS - 1)) * STRIP) * 4u);
                sq1[d] = lds128v(sim_lane + (uint32_t)(((r + 1) & (SIM_ROWS - 1)) * STRIP) * 4u);
                bq0[d] = lds32v(st.bnd_base + 4u * ((RPS * s) & (BND_RING - 1)));
                bq1[d] = lds32v(st.bnd_base + 4u * ((RPS * s + 1) & (BND_RING - 1)));
            }
#pragma unroll
            for (int u = 0; u < TILE / RPS; ++u) {
                const int s = k * (TILE / RPS) + u;
                const int r0 = RPS * (s - lane);         // this lane's two rows r0, r0 + 1
                if (u % (BATCH / RPS) == 0) {
                    // lane 0 needs batch b = s / 4 from step 4b; commit b + 1 now, issue b + 2
                    const int b = s / (BATCH / RPS);
                    if (b + 1 < nbatches) bnd_commit(st, b + 1, bnd_pending);
                    bnd_pending = b + 2 < nbatches ? bnd_issue(st, b + 2) : 0;
                }
                const int4 a = sq0[u % PF], c = sq1[u % PF];
                const int b0 = bq0[u % PF], b1 = bq1[u % PF];
                sq0[u % PF] = lds128v(sim_lane + (uint32_t)(((r0 + RPS * PF) & (SIM_ROWS - 1)) * STRIP) * 4u);
                sq1[u % PF] = lds128v(sim_lane + (uint32_t)(((r0 + RPS * PF + 1) & (SIM_ROWS - 1)) * STRIP) * 4u);
                bq0[u % PF] = lds32v(st.bnd_base + 4u * ((RPS * (s + PF)) & (BND_RING - 1)));
                bq1[u % PF] = lds32v(st.bnd_base + 4u * ((RPS * (s + PF) + 1) & (BND_RING - 1)));
                // row r0: left-independent parts first (overlap the shuffles)
                const int x0 = max(left_prev + a.x, h0 - p);
                const int x1 = max(h0 + a.y, h1 - p);
                const int x2 = max(h1 + a.z, h2 - p);
                const int x3 = max(h2 + a.w, h3 - p);
                // lane j-1 finished rows r0, r0 + 1 in the previous step
                const int sl0 = __shfl_up_sync(0xffffffffu, t3, 1);
                const int sl1 = __shfl_up_sync(0xffffffffu, h3, 1);
                const int left0 = lane == 0 ? b0 : sl0;
                const int left1 = lane == 0 ? b1 : sl1;
                const int v0 = max(left0 - p, x0);
                const int v1 = max(v0 - p, x1);
                const int v2 = max(v1 - p, x2);
                const int v3 = max(v2 - p, x3);
                // row r0 + 1: up = row r0, diagonal of its first cell = row r0's left value
                const int w0 = max(max(left0 + c.x, v0 - p), left1 - p);
                const int w1 = max(max(v0 + c.y, v1 - p), w0 - p);
                const int w2 = max(max(v1 + c.z, v2 - p), w1 - p);
                const int w3 = max(max(v2 + c.w, v3 - p), w2 - p);
                if (k > 1 || r0 >= 0) {                  // lanes start one step apart (the
                    // 31-step skew spans the first two 16-step blocks)
                    out_ring[(r0 & (OUT_ROWS - 1)) * (STRIP / 4)] = make_int4(v0, v1, v2, v3);
                    out_ring[((r0 + 1) & (OUT_ROWS - 1)) * (STRIP / 4)] = make_int4(w0, w1, w2, w3);
                    h0 = w0; h1 = w1; h2 = w2; h3 = w3; t3 = v3;
                    left_prev = left1;
                    // the strip's last column goes straight to the right neighbour
                    if (lane == 31 && r0 < n) {
                        const unsigned long long e0 =
                            ((unsigned long long)(st.tag | (unsigned)(r0 + 1)) << 32) | (unsigned)v3;
                        asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" :: "l"(st.my_bnd2 + r0), "l"(e0)
                                     : "memory");
                        if (r0 + 1 < n) {
                            const unsigned long long e1 =
                                ((unsigned long long)(st.tag | (unsigned)(r0 + 2)) << 32) | (unsigned)w3;
                            asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" :: "l"(st.my_bnd2 + r0 + 1),
                                         "l"(e1) : "memory");
                        }
                    }
                }
            }
        }
        cp_async_wait_all();
        __syncwarp();
    }
}

}  // namespace

extern "C" lego_status lego_nw_i32(const int32_t* sim, int32_t* score, int64_t n, int32_t penalty, int64_t batch,
                                   void* stream) {
    if (n < 0 || batch < 0) return lego_fail(LEGO_E_SHAPE, "negative NW size");
    if (batch == 0) return LEGO_OK;
    if (n > (1 << 20)) return lego_fail(LEGO_E_SHAPE, "NW n above 2^20");
    if (!sim || !score) return lego_fail(LEGO_E_ARG, "null buffer");
    if ((uintptr_t)sim & 15) return lego_fail(LEGO_E_ARG, "sim must be 16-byte aligned");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const long long w = n + 1;
    const long long bgrid = (batch * w + 255) / 256;
    nw_borders<<<(unsigned)(bgrid < 4096 ? bgrid : 4096), 256, 0, st>>>(score, n, penalty, batch);
    if (n == 0) return lego_cuda_check(cudaGetLastError(), "nw borders");
    const int strips = (int)((n + STRIP - 1) / STRIP);
    const long long total = (long long)strips * batch;
    if (total > INT32_MAX) return lego_fail(LEGO_E_SHAPE, "NW batch too large");
    const int n_pad = (int)((n + TILE - 1) / TILE * TILE);
    const size_t bnd_off = 256;
    const size_t bnd_bytes = sizeof(int2) * (size_t)total * n_pad;
    char* scratch = nullptr;
    LEGO_TRY(lego_cuda_check(cudaMallocAsync((void**)&scratch, bnd_off + bnd_bytes, st), "cudaMallocAsync"));
    // ticket + tagged boundary words start at zero; tags also carry a launch epoch
    LEGO_TRY(lego_cuda_check(cudaMemsetAsync(scratch, 0, bnd_off + bnd_bytes, st), "cudaMemsetAsync"));
    int* ticket = reinterpret_cast<int*>(scratch);
    int2* bnd2 = reinterpret_cast<int2*>(scratch + bnd_off);
    static unsigned epoch = 0;
    epoch = (epoch + 1) & 0x7FFu;
    if (epoch == 0) epoch = 1;
    static cudaError_t attr = cudaFuncSetAttribute(nw_strips, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   SMEM_BYTES);
    LEGO_TRY(lego_cuda_check(attr, "cudaFuncSetAttribute(nw)"));
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const long long cap = 2LL * sms;       // two strips per SM fit the staging rings
    const long long ctas = total < cap ? total : cap;
    nw_strips<<<(unsigned)ctas, 32, SMEM_BYTES, st>>>(sim, score, (int)n, penalty, strips, (int)total, ticket,
                                                      bnd2, epoch);
    lego_status s = lego_cuda_check(cudaGetLastError(), "nw launch");
    cudaFreeAsync(scratch, st);
    return s;
}
