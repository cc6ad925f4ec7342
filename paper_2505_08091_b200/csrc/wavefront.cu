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
//  * inside a strip the warp sweeps anti-diagonally: lane j owns columns
//    4j..4j+3 and at step s computes row s - j, i.e. every step is one
//    anti-diagonal of the (rows x 32 lane-columns) grid -- the LEGO antidiag
//    order of the paper's NW kernel.  The value from the
//    left arrives by warp shuffle, the up and diagonal values are the lane's
//    own previous row: the per-step critical path is one shuffle plus a
//    4-cell max/add chain.  Everything else is off that path:
//  * sim is staged 32 rows x 128 columns at a time by cp.async two blocks
//    ahead (4 buffers) and each lane's next 16-byte sim vector is read from
//    shared memory one step early;
//  * results go through a 32 x 128 tile and leave as coalesced row segments
//    once a block of 32 rows is complete; at that point the strip's last
//    column for those rows is copied to a global boundary array and
//    published with one st.release, which the right neighbour polls with
//    ld.acquire once per 32 rows.
#include <cuda_runtime.h>

#include <cstdint>

#include "lego_common.h"

namespace {

constexpr int TILE = 32;                 // rows per staged block
constexpr int CPL = 4;                   // columns per lane
constexpr int STRIP = 32 * CPL;          // columns per warp strip
constexpr int SIM_BUFS = 4;
constexpr int OUT_BUFS = 2;
constexpr int BLOCK_ELEMS = TILE * STRIP;
constexpr int BND_RING = 64;
constexpr int SMEM_BYTES = (SIM_BUFS + OUT_BUFS) * BLOCK_ELEMS * 4 + BND_RING * 4;

__device__ __forceinline__ void st_release(int* p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;"
                 :: "r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst))), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;"
                 :: "r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst))), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

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

// stage sim rows [32k, 32k+32) of the strip into buf (one cp.async group; empty past the end)
__device__ __forceinline__ void stage_sim(int32_t* buf, const int32_t* simb, int n, int k, int col0, int lane,
                                          bool vec_ok) {
    for (int r = 0; r < TILE; ++r) {
        const int row = k * TILE + r;
        if (row >= n) break;
        const int32_t* src = simb + (long long)row * n + col0;
        int32_t* dst = buf + r * STRIP;
        if (vec_ok) {
            if (col0 + CPL * lane < n) cp_async16(dst + CPL * lane, src + CPL * lane);
        } else {
#pragma unroll
            for (int q = 0; q < CPL; ++q) {
                const int c = q * 32 + lane;
                if (col0 + c < n) cp_async4(dst + c, src + c);
            }
        }
    }
    cp_async_commit();
}

__global__ void __launch_bounds__(32)
nw_strips(const int32_t* __restrict__ sim, int32_t* __restrict__ score, int n, int p, int strips_per_matrix,
          int total_strips, int* __restrict__ ticket, int* __restrict__ progress, int32_t* __restrict__ bnd) {
    extern __shared__ __align__(16) int32_t smem[];
    int32_t* s_sim = smem;                                   // [4][32][128]
    int32_t* s_out = s_sim + SIM_BUFS * BLOCK_ELEMS;         // [2][32][128]
    int32_t* s_bnd = s_out + OUT_BUFS * BLOCK_ELEMS;         // ring of 64 rows
    const int lane = threadIdx.x;
    const long long ld = (long long)n + 1;
    const int n_pad = (n + TILE - 1) / TILE * TILE;
    const int nblocks = n_pad / TILE;
    const bool vec_ok = (n % 4) == 0;

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
        const int32_t* left_bnd = my_bnd - n_pad;
        int* my_prog = progress + strip;
        const int* left_prog = progress + strip - 1;
        const int col0 = w * STRIP;
        const int c_lane = col0 + CPL * lane;                 // first 0-based sim column of this lane

        // block boundary event for block k: its sim landed, block k+1 in flight,
        // left boundary rows of block k in the ring
        auto enter_block = [&](int k) {
            if (k + 1 < nblocks) {
                stage_sim(s_sim + ((k + 1) & (SIM_BUFS - 1)) * BLOCK_ELEMS, simb, n, k + 1, col0, lane, vec_ok);
                cp_async_wait_1();
            } else {
                cp_async_wait_all();
            }
            if (w > 0) {
                const int need = min((k + 1) * TILE, n);
                if (lane == 0) {
                    // relaxed polling (no L1 invalidation per probe), one acquire at the end
                    while (*reinterpret_cast<const volatile int*>(left_prog) < need) {
                    }
                    (void)ld_acquire(left_prog);
                }
                __syncwarp();
                const int row = k * TILE + lane;
                if (row < n) s_bnd[row & (BND_RING - 1)] = __ldcg(left_bnd + row);
            }
            __syncwarp();
        };

        stage_sim(s_sim, simb, n, 0, col0, lane, vec_ok);
        enter_block(0);

        int32_t h[CPL];
#pragma unroll
        for (int k = 0; k < CPL; ++k) h[k] = -(c_lane + k + 1) * p;   // S[0][c+1]
        int32_t left_prev = -c_lane * p;                               // S[0][c_lane]
        int4 sv = make_int4(0, 0, 0, 0);
        if (lane == 0) sv = *reinterpret_cast<const int4*>(s_sim);    // row 0 for lane 0

        for (int s = 0; s < n_pad + TILE - 1; ++s) {
            const int i = s - lane;
            int32_t left = __shfl_up_sync(0xffffffffu, h[CPL - 1], 1);   // S[i+1][c_lane] from lane-1
            if (lane == 0) left = w == 0 ? -(i + 1) * p : s_bnd[i & (BND_RING - 1)];
            if (i >= 0 && i < n) {
                const int32_t svals[CPL] = {sv.x, sv.y, sv.z, sv.w};
                int32_t diag = left_prev, lf = left;
#pragma unroll
                for (int k = 0; k < CPL; ++k) {
                    const int32_t v = max(diag + svals[k], max(h[k], lf) - p);
                    diag = h[k];
                    h[k] = v;
                    lf = v;
                }
                *reinterpret_cast<int4*>(s_out + ((i >> 5) & 1) * BLOCK_ELEMS + (i & (TILE - 1)) * STRIP +
                                         CPL * lane) = make_int4(h[0], h[1], h[2], h[3]);
            }
            left_prev = left;
            // block k completes at step 32k + 62: publish the boundary column first (the
            // release must not wait behind the row stores), then flush the rows
            if ((s & (TILE - 1)) == TILE - 2 && s >= 2 * TILE - 2) {
                const int k = (s - (2 * TILE - 2)) / TILE;
                __syncwarp();
                const int32_t* src = s_out + (k & 1) * BLOCK_ELEMS;
                const int brow = k * TILE + lane;
                if (brow < n) my_bnd[brow] = src[lane * STRIP + STRIP - 1];
                __threadfence();                     // each lane's boundary value is visible GPU-wide
                __syncwarp();
                if (lane == 0) st_release(my_prog, min((k + 1) * TILE, n));
                for (int r = 0; r < TILE; ++r) {
                    const int row = k * TILE + r;
                    if (row >= n) break;
                    int32_t* dst = sc + (long long)(row + 1) * ld + col0 + 1;
#pragma unroll
                    for (int q = 0; q < CPL; ++q) {
                        const int c = q * 32 + lane;
                        if (col0 + c < n) dst[c] = src[r * STRIP + c];
                    }
                }
                __syncwarp();
            }
            // next step reads row i + 1; a new block enters when lane 0 crosses into it
            if (((s + 1) & (TILE - 1)) == 0 && (s + 1) < n_pad) enter_block((s + 1) / TILE);
            const int ni = i + 1;
            if (ni >= 0 && ni < n)
                sv = *reinterpret_cast<const int4*>(s_sim + ((ni >> 5) & (SIM_BUFS - 1)) * BLOCK_ELEMS +
                                                    (ni & (TILE - 1)) * STRIP + CPL * lane);
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
    const long long cap = 2LL * sms;       // two strips per SM fit the staging buffers
    const long long ctas = total < cap ? total : cap;
    nw_strips<<<(unsigned)ctas, 32, SMEM_BYTES, st>>>(sim, score, (int)n, penalty, strips, (int)total, ticket,
                                                      progress, bnd);
    lego_status s = lego_cuda_check(cudaGetLastError(), "nw launch");
    cudaFreeAsync(scratch, st);
    return s;
}
