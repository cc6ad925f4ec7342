// wavefront.cu -- Needleman-Wunsch score matrix as an anti-diagonal wavefront
// (BASELINE.json config 4b).
//
//   S[0][j] = -j*p,  S[i][0] = -i*p,
//   S[i][j] = max(S[i-1][j-1] + sim[i-1][j-1], S[i-1][j] - p, S[i][j-1] - p)
//
// Decomposition (B200-first, no host loop over diagonals): the n columns are
// cut into 32-wide strips, one warp per strip, claimed in order from an
// atomic ticket so a strip's left neighbour is always already running (no
// deadlock, no grid sync).  Inside a strip the warp sweeps the strip's cells
// in anti-diagonal order: lane j owns column j and at step s computes row
// s - j, so each step is one anti-diagonal of the 32-wide strip (the LEGO
// antidiag order of the paper's NW kernel).  The left
// neighbour's value arrives by warp shuffle, the up value is the lane's own
// previous result, the diagonal value is the previous shuffle.  sim rows are
// staged 32x32 through shared memory with coalesced loads (prefetched one
// block ahead) and read back along the anti-diagonal -- bank = lane, no
// conflicts; results go through a second 32x32 tile and leave as coalesced
// row segments.  Strips hand their last column to the right neighbour
// through a global boundary array published every 32 rows with st.release /
// ld.acquire.
#include <cuda_runtime.h>

#include <cstdint>

#include "lego_common.h"

namespace {

constexpr int WARPS = 8;
constexpr int TILE = 32;

__device__ __forceinline__ void st_release(int* p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
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

__global__ void __launch_bounds__(WARPS * 32)
nw_strips(const int32_t* __restrict__ sim, int32_t* __restrict__ score, int n, int p, int strips_per_matrix,
          int total_strips, int* __restrict__ ticket, int* __restrict__ progress, int32_t* __restrict__ bnd) {
    extern __shared__ int32_t smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int32_t* s_sim = smem + warp * (4 * TILE * TILE);      // [2][32][32]
    int32_t* s_out = s_sim + 2 * TILE * TILE;              // [2][32][32]
    const long long ld = (long long)n + 1;
    const int n_pad = (n + TILE - 1) / TILE * TILE;
    const int nblocks = n_pad / TILE;

    for (;;) {
        int strip = 0;
        if (lane == 0) strip = atomicAdd(ticket, 1);
        strip = __shfl_sync(0xffffffffu, strip, 0);
        if (strip >= total_strips) return;
        const int b = strip / strips_per_matrix;
        const int w = strip - b * strips_per_matrix;
        const int32_t* simb = sim + (long long)b * n * n;
        int32_t* sc = score + (long long)b * ld * ld;
        int32_t* my_bnd = bnd + (long long)strip * n_pad;
        const int32_t* left_bnd = my_bnd - n_pad;          // strip - 1 (same matrix when w > 0)
        int* my_prog = progress + strip;
        const int* left_prog = progress + strip - 1;
        const int col = w * TILE + lane;                  // 0-based sim column; DP column col + 1
        const bool col_ok = col < n;

        // prefetch sim block 0 (rows 0..31 of this strip), coalesced per row
        int32_t pre[TILE];
#pragma unroll
        for (int r = 0; r < TILE; ++r) pre[r] = (r < n && col_ok) ? __ldg(simb + (long long)r * n + col) : 0;

        int32_t h = -(col + 1) * p;                        // S[0][col+1] until the lane starts
        int32_t left_prev = -col * p;                      // S[0][col]
        int known = 0;                                     // rows published by the left strip
        int32_t lane0_diag = -(w * TILE) * p;              // S[i][w*32] for lane 0

        for (int s = 0; s < n_pad + TILE - 1; ++s) {
            if ((s & (TILE - 1)) == 0) {
                const int k = s / TILE;
                if (k < nblocks) {
                    int32_t* dst = s_sim + (k & 1) * TILE * TILE;
#pragma unroll
                    for (int r = 0; r < TILE; ++r) dst[r * TILE + lane] = pre[r];
                    const int nk = k + 1;
                    if (nk < nblocks) {
#pragma unroll
                        for (int r = 0; r < TILE; ++r) {
                            const int row = nk * TILE + r;
                            pre[r] = (row < n && col_ok) ? __ldg(simb + (long long)row * n + col) : 0;
                        }
                    }
                }
                __syncwarp();
            }
            const int i = s - lane;                        // 0-based row of this lane at step s
            int32_t from_left = __shfl_up_sync(0xffffffffu, h, 1);   // S[i+1][col] from lane-1
            if (lane == 0) {
                if (w == 0) {
                    from_left = -(i + 1) * p;
                } else if (i < n) {
                    if (i >= known) {
                        do { known = ld_acquire(left_prog); } while (known <= i);
                    }
                    from_left = __ldcg(left_bnd + i);
                }
            }
            const bool active = i >= 0 && i < n;
            if (active) {
                const int32_t sv = s_sim[((i / TILE) & 1) * TILE * TILE + (i & (TILE - 1)) * TILE + lane];
                const int32_t diag = lane == 0 ? lane0_diag : left_prev;
                const int32_t up = h;
                int32_t v = diag + sv;
                const int32_t g = max(up, from_left) - p;
                h = max(v, g);
                s_out[((i / TILE) & 1) * TILE * TILE + (i & (TILE - 1)) * TILE + lane] = h;
                if (lane == TILE - 1) {
                    my_bnd[i] = h;
                    if ((i & (TILE - 1)) == TILE - 1 || i == n - 1) st_release(my_prog, i + 1);
                }
            }
            if (lane == 0) lane0_diag = from_left;
            left_prev = from_left;
            // block k completes at step 32k + 62: flush its 32 rows as coalesced segments
            if ((s & (TILE - 1)) == TILE - 2 && s >= 2 * TILE - 2) {
                const int k = (s - (2 * TILE - 2)) / TILE;
                __syncwarp();
                const int32_t* src = s_out + (k & 1) * TILE * TILE;
                for (int r = 0; r < TILE; ++r) {
                    const int row = k * TILE + r;
                    if (row < n && col_ok) sc[(long long)(row + 1) * ld + col + 1] = src[r * TILE + lane];
                }
                __syncwarp();
            }
        }
    }
}

}  // namespace

extern "C" lego_status lego_nw_i32(const int32_t* sim, int32_t* score, int64_t n, int32_t penalty, int64_t batch,
                                   void* stream) {
    if (n < 0 || batch < 0) return lego_fail(LEGO_E_SHAPE, "negative NW size");
    if (batch == 0) return LEGO_OK;
    if (n > (1 << 20)) return lego_fail(LEGO_E_SHAPE, "NW n above 2^20");
    if (!sim || !score) return lego_fail(LEGO_E_ARG, "null buffer");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const long long w = n + 1;
    nw_borders<<<(unsigned)((batch * w + 255) / 256 < 4096 ? (batch * w + 255) / 256 : 4096), 256, 0, st>>>(
        score, n, penalty, batch);
    if (n == 0) return lego_cuda_check(cudaGetLastError(), "nw borders");
    const int strips = (int)((n + TILE - 1) / TILE);
    const long long total = (long long)strips * batch;
    if (total > INT32_MAX) return lego_fail(LEGO_E_SHAPE, "NW batch too large");
    const int n_pad = strips * TILE;
    // scratch: ticket + per-strip progress + boundary columns
    const size_t prog_bytes = sizeof(int) * (size_t)(total + 1);
    const size_t bnd_bytes = sizeof(int32_t) * (size_t)total * n_pad;
    char* scratch = nullptr;
    LEGO_TRY(lego_cuda_check(cudaMallocAsync((void**)&scratch, prog_bytes + bnd_bytes, st), "cudaMallocAsync"));
    LEGO_TRY(lego_cuda_check(cudaMemsetAsync(scratch, 0, prog_bytes, st), "cudaMemsetAsync"));
    int* ticket = reinterpret_cast<int*>(scratch);
    int* progress = ticket + 1;
    int32_t* bnd = reinterpret_cast<int32_t*>(scratch + prog_bytes);
    const int smem = WARPS * 4 * TILE * TILE * (int)sizeof(int32_t);
    static cudaError_t attr = cudaFuncSetAttribute(nw_strips, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    LEGO_TRY(lego_cuda_check(attr, "cudaFuncSetAttribute(nw)"));
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    long long ctas = (total + WARPS - 1) / WARPS;
    if (ctas > 2LL * sms) ctas = 2LL * sms;
    nw_strips<<<(unsigned)ctas, WARPS * 32, smem, st>>>(sim, score, (int)n, penalty, strips, (int)total, ticket,
                                                        progress, bnd);
    lego_status s = lego_cuda_check(cudaGetLastError(), "nw launch");
    cudaFreeAsync(scratch, st);
    return s;
}
