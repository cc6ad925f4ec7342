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
//  * a strip is two 64-column *chains*; in chain g lane j owns columns
//    64g + 2j, 64g + 2j + 1 and at warp step s computes row s - 32g - j:
//    every step advances one anti-diagonal of each chain (the LEGO antidiag
//    order of the paper's NW kernel).  The left value
//    arrives by a rotating warp shuffle: lane j reads lane j-1, lane 0 reads
//    lane 31, which sends chain g-1's last column (computed one step
//    earlier) or, for chain 0, the left strip's boundary value.  The two
//    chains are independent within a step, so each one's shuffle latency is
//    hidden behind the other's work; up and diagonal values are the lane's
//    own previous row;
//  * sim is staged 32 rows x 128 columns at a time by cp.async one block
//    ahead into a 128-row ring and read from shared memory four steps ahead
//    (register queue); results go to a 128-row ring and leave as coalesced
//    row segments once a block of rows is complete, when the strip's last
//    column is also published to a global boundary array with one
//    st.release (polled by the right neighbour once per 32 rows).
#include <cuda_runtime.h>

#include <cstdint>

#include "lego_common.h"

namespace {

constexpr int TILE = 32;                 // rows per block
constexpr int CHAINS = 2;                // independent chains per warp
constexpr int CPL = 2;                   // columns per lane per chain
constexpr int CHAIN_COLS = 32 * CPL;     // 64
constexpr int STRIP = CHAINS * CHAIN_COLS;   // 128 columns per warp
constexpr int RING = 128;                // rows in the sim ring and in the out ring
constexpr int BND_RING = 64;
constexpr int LAG = TILE * (CHAINS - 1) + 31;   // steps from chain 0 lane 0 to the last cell of a row
constexpr int SMEM_BYTES = 2 * RING * STRIP * 4 + BND_RING * 4;
constexpr int PF = 4;                    // sim prefetch distance (steps)

__device__ __forceinline__ void st_release(int* p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async4(uint32_t dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" :: "r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
__device__ __forceinline__ int2 lds64v(uint32_t a) {
    int2 v;
    asm volatile("ld.shared.v2.b32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
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
    int32_t* my_bnd;
    const int32_t* left_bnd;
    int* my_prog;
    const int* left_prog;
    int n, p, w, col0, lane;
    bool vec_ok;
    uint32_t sim_base, out_base, bnd_base;   // shared-window addresses
    int32_t* out_gen;                        // generic pointer of the out ring
};

// stage sim rows [32k, 32k+32) of the strip into the ring (one cp.async group)
__device__ __forceinline__ void stage_sim(const Strip& st, int k) {
    const int rows = min(TILE, st.n - k * TILE);
    uint32_t dst = st.sim_base + (uint32_t)(((k * TILE) & (RING - 1)) * STRIP) * 4u;
    if (st.vec_ok) {
        const int32_t* src = st.simb + (long long)k * TILE * st.n + st.col0 + 4 * st.lane;
        const bool ok = st.col0 + 4 * st.lane < st.n;
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
            for (int q = 0; q < STRIP / 32; ++q)
                if (st.col0 + q * 32 + st.lane < st.n) cp_async4(dst + 128u * q, src + 32 * q);
            dst += STRIP * 4u;
            src += st.n;
        }
    }
    cp_async_commit();
}

// block k enters (chain 0 lane 0 reaches row 32k): sim block k landed, block
// k+1 in flight, left boundary rows of block k in the ring
__device__ __forceinline__ void enter_block(const Strip& st, int k, int nblocks) {
    if (k + 1 < nblocks) {
        stage_sim(st, k + 1);
        cp_async_wait_1();
    } else {
        cp_async_wait_all();
    }
    const int row = k * TILE + st.lane;
    int32_t v;
    if (st.w > 0) {
        const int need = min((k + 1) * TILE, st.n);
        if (st.lane == 0) {
            while (*reinterpret_cast<const volatile int*>(st.left_prog) < need) {
            }
            (void)ld_acquire(st.left_prog);
        }
        __syncwarp();
        v = row < st.n ? __ldcg(st.left_bnd + row) : 0;
    } else {
        v = -(row + 1) * st.p;               // S[row+1][0]
    }
    asm volatile("st.shared.b32 [%0], %1;" :: "r"(st.bnd_base + 4u * (row & (BND_RING - 1))), "r"(v)
                 : "memory");
    __syncwarp();
}

// block k is complete: publish its boundary column, then write its rows out
__device__ __forceinline__ void flush_block(const Strip& st, int k) {
    __syncwarp();
    const int32_t* src = st.out_gen + ((k * TILE) & (RING - 1)) * STRIP;
    const int brow = k * TILE + st.lane;
    if (brow < st.n) st.my_bnd[brow] = src[st.lane * STRIP + STRIP - 1];
    __threadfence();
    __syncwarp();
    if (st.lane == 0) st_release(st.my_prog, min((k + 1) * TILE, st.n));
    const long long ld = (long long)st.n + 1;
    const int rows = min(TILE, st.n - k * TILE);
    int32_t* dst = st.sc + (long long)(k * TILE + 1) * ld + st.col0 + 1 + st.lane;
    const int32_t* s = src + st.lane;
    bool ok[STRIP / 32];
#pragma unroll
    for (int q = 0; q < STRIP / 32; ++q) ok[q] = st.col0 + q * 32 + st.lane < st.n;
#pragma unroll 8
    for (int r = 0; r < rows; ++r) {
#pragma unroll
        for (int q = 0; q < STRIP / 32; ++q)
            if (ok[q]) dst[32 * q] = s[32 * q];
        dst += ld;
        s += STRIP;
    }
    __syncwarp();
}

__global__ void __launch_bounds__(32)
nw_strips(const int32_t* __restrict__ sim, int32_t* __restrict__ score, int n, int p, int strips_per_matrix,
          int total_strips, int* __restrict__ ticket, int* __restrict__ progress, int32_t* __restrict__ bnd) {
    extern __shared__ __align__(16) int32_t smem[];
    const int lane = threadIdx.x;
    const int n_pad = (n + TILE - 1) / TILE * TILE;
    const int nblocks = n_pad / TILE;
    Strip st;
    st.n = n;
    st.p = p;
    st.lane = lane;
    st.vec_ok = (n % 4) == 0;
    st.sim_base = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
    st.out_base = st.sim_base + RING * STRIP * 4;
    st.bnd_base = st.out_base + RING * STRIP * 4;
    st.out_gen = smem + RING * STRIP;
    // per-lane byte offsets of chain g's two columns inside a ring row
    const uint32_t lane_off0 = 4u * (CPL * lane);
    const uint32_t lane_off1 = 4u * (CHAIN_COLS + CPL * lane);

    for (;;) {
        int strip = 0;
        if (lane == 0) strip = atomicAdd(ticket, 1);
        strip = __shfl_sync(0xffffffffu, strip, 0);
        if (strip >= total_strips) return;
        const int b = strip / strips_per_matrix;
        st.w = strip - b * strips_per_matrix;
        st.simb = sim + (long long)b * n * n;
        st.sc = score + (long long)b * ((long long)n + 1) * ((long long)n + 1);
        st.my_bnd = bnd + (long long)strip * n_pad;
        st.left_bnd = st.my_bnd - n_pad;
        st.my_prog = progress + strip;
        st.left_prog = progress + strip - 1;
        st.col0 = st.w * STRIP;
        // 0-based sim column of the first column this lane owns in chain 0 / chain 1
        const int c0 = st.col0 + CPL * lane, c1 = c0 + CHAIN_COLS;

        stage_sim(st, 0);
        // h: the lane's two cells of the previous row (S[0][c+1], S[0][c+2] to start)
        int a0 = -(c0 + 1) * p, a1 = -(c0 + 2) * p;       // chain 0
        int b0 = -(c1 + 1) * p, b1 = -(c1 + 2) * p;       // chain 1
        int la = -c0 * p, lb = -c1 * p;                    // S[i][c] of the cell left of each chain's lane

        // blocks enter while chain 0 needs them; the extra iterations drain chain 1 and the flushes
        const int last_iter = nblocks + (LAG + TILE - 1) / TILE + 1;
        for (int k = 0; k <= last_iter; ++k) {
            if (k >= 3) flush_block(st, k - 3);            // block k-3 completed at step 32k - 2
            if (k >= last_iter) break;
            if (k < nblocks) enter_block(st, k, nblocks);
            // operand queues, PF steps ahead; refilled at every block start because
            // reads past the entering block may have seen unlanded rows
            int2 qa[PF], qb[PF];
            int qbv[PF];
#pragma unroll
            for (int d = 0; d < PF; ++d) {
                const int s = k * TILE + d;
                qa[d] = lds64v(st.sim_base + (uint32_t)(((s - lane) & (RING - 1)) * STRIP) * 4u + lane_off0);
                qb[d] = lds64v(st.sim_base + (uint32_t)(((s - TILE - lane) & (RING - 1)) * STRIP) * 4u + lane_off1);
                qbv[d] = lds32v(st.bnd_base + 4u * (s & (BND_RING - 1)));
            }
#pragma unroll
            for (int u = 0; u < TILE; ++u) {
                const int s = k * TILE + u;
                const int ia = s - lane;                   // chain 0 row of this lane
                const int ib = ia - TILE;                  // chain 1 row of this lane
                const int2 sa = qa[u % PF], sb = qb[u % PF];
                const int bv = qbv[u % PF];
                qa[u % PF] = lds64v(st.sim_base + (uint32_t)(((ia + PF) & (RING - 1)) * STRIP) * 4u + lane_off0);
                qb[u % PF] = lds64v(st.sim_base + (uint32_t)(((ib + PF) & (RING - 1)) * STRIP) * 4u + lane_off1);
                qbv[u % PF] = lds32v(st.bnd_base + 4u * ((s + PF) & (BND_RING - 1)));
                // left-independent parts: x_c = max(diag_c + sim_c, up_c - p)
                const int xa0 = max(la + sa.x, a0 - p), xa1 = max(a0 + sa.y, a1 - p);
                const int xb0 = max(lb + sb.x, b0 - p), xb1 = max(b0 + sb.y, b1 - p);
                // rotating shuffle: lane 31 feeds lane 0 -- chain 0 gets the left strip's
                // boundary, chain 1 gets chain 0's last column of the previous step
                const int sa_send = lane == 31 ? bv : a1;
                const int sb_send = lane == 31 ? a1 : b1;
                const int left_a = __shfl_sync(0xffffffffu, sa_send, (lane + 31) & 31);
                const int left_b = __shfl_sync(0xffffffffu, sb_send, (lane + 31) & 31);
                const int va0 = max(left_a - p, xa0), va1 = max(va0 - p, xa1);
                const int vb0 = max(left_b - p, xb0), vb1 = max(vb0 - p, xb1);
                if (ia >= 0) { a0 = va0; a1 = va1; la = left_a; }     // lanes start one step apart,
                if (ib >= 0) { b0 = vb0; b1 = vb1; lb = left_b; }     // chain 1 one block later
                if ((unsigned)ia < (unsigned)n)
                    *reinterpret_cast<int2*>(st.out_gen + (ia & (RING - 1)) * STRIP + CPL * lane) = make_int2(a0, a1);
                if ((unsigned)ib < (unsigned)n)
                    *reinterpret_cast<int2*>(st.out_gen + (ib & (RING - 1)) * STRIP + CHAIN_COLS + CPL * lane) =
                        make_int2(b0, b1);
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
    const size_t prog_bytes = sizeof(int) * (size_t)(total + 1);
    const size_t bnd_off = (prog_bytes + 255) / 256 * 256;
    const size_t bnd_bytes = sizeof(int32_t) * (size_t)total * n_pad;
    char* scratch = nullptr;
    LEGO_TRY(lego_cuda_check(cudaMallocAsync((void**)&scratch, bnd_off + bnd_bytes, st), "cudaMallocAsync"));
    LEGO_TRY(lego_cuda_check(cudaMemsetAsync(scratch, 0, prog_bytes, st), "cudaMemsetAsync"));
    int* ticket = reinterpret_cast<int*>(scratch);
    int* progress = ticket + 1;
    int32_t* bnd = reinterpret_cast<int32_t*>(scratch + bnd_off);
    static cudaError_t attr = cudaFuncSetAttribute(nw_strips, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   SMEM_BYTES);
    LEGO_TRY(lego_cuda_check(attr, "cudaFuncSetAttribute(nw)"));
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const long long ctas = total < sms ? total : sms;      // one strip-warp per SM (128 KiB staging)
    nw_strips<<<(unsigned)ctas, 32, SMEM_BYTES, st>>>(sim, score, (int)n, penalty, strips, (int)total, ticket,
                                                      progress, bnd);
    lego_status s = lego_cuda_check(cudaGetLastError(), "nw launch");
    cudaFreeAsync(scratch, st);
    return s;
}
