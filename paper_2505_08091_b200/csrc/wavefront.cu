// wavefront.cu -- Needleman-Wunsch score matrix as an anti-diagonal wavefront
// (BASELINE.json config 4b).
//
//   S[0][j] = -j*p,  S[i][0] = -i*p,
//   S[i][j] = max(S[i-1][j-1] + sim[i-1][j-1], S[i-1][j] - p, S[i][j-1] - p)
//
// Offset scores.  With S'[i][j] = S[i][j] + (i+j)*p the recurrence becomes
//   S'[i][j] = max(S'[i-1][j-1] + sim[i-1][j-1] + 2p, S'[i-1][j], S'[i][j-1])
// with all-zero borders: the left-to-right dependency chain is one integer
// max per cell (no subtract), and the conversion back to S happens in the
// store path, off the chain.  Exact whenever |p|*(2n+2) < 2^30 and the true
// scores fit in +-2^30 (checked on p; sim is the caller's contract).
//
// Decomposition (no host loop over diagonals, no grid sync):
//  * the n columns are cut into 128-wide strips, one CTA per strip, claimed in
//    order from an atomic ticket (a strip's left neighbour is always already
//    running); a persistent grid of at most one CTA per SM;
//  * four warp roles per CTA, one per SM sub-partition:
//      warp 0  compute:  sweeps the strip anti-diagonally over 2x4 cell blocks
//              -- lane j owns columns 4j..4j+3 and at step s computes rows
//              2(s-j), 2(s-j)+1, i.e. each step is one anti-diagonal of the
//              (row pairs x 32 lane-columns) grid, the LEGO antidiag order of
//              the paper's NW kernel.  The two left
//              values arrive by one warp shuffle each; everything else is in
//              registers or one 16-byte shared load;
//      warp 1  producer: cp.async-stages sim, 32 rows x 128 columns per
//              block, into an 8-block ring (the compute warp overwrites each
//              sim row with its S' row in place);
//      warp 2  boundary: polls the left strip's published last column
//              (tagged 64-bit words in global memory: value | launch epoch |
//              row) and deposits it, tagged with the row, in a shared ring
//              that compute lane 0 reads one step ahead;
//      warp 3  flusher:  converts finished blocks S' -> S and writes them
//              out as coalesced row segments;
//  * roles synchronise through monotonic block counters in shared memory
//    (loaded / computed / flushed); the compute warp checks them once per
//    32 rows with a prefetched load, so its step body has no barrier.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <utility>

#include "lego_common.h"

namespace {

constexpr int CPL = 4;                               // columns per lane
constexpr int STRIP = 32 * CPL;                      // columns per strip
constexpr int BLK = 32;                              // rows per block
constexpr int STEPS = BLK / 2;                       // compute steps per block
constexpr int NSLOT = 8;                             // ring blocks
constexpr int RING_ROWS = NSLOT * BLK;               // 256
constexpr int ROW_BYTES = STRIP * 4;                 // 512
constexpr int RING_BYTES = RING_ROWS * ROW_BYTES;    // 128 KiB
constexpr int BND_BYTES = RING_ROWS * 4;
constexpr int CTRL_BYTES = 64;
constexpr int SMEM_BYTES = RING_BYTES + BND_BYTES + CTRL_BYTES;
#ifndef NW_POLL_NS
#define NW_POLL_NS 32                                // boundary poll back-off
#endif
constexpr int DRAIN = 2;                             // 32 extra steps cover lane 31's 31-step lag

#ifdef LEGO_NW_DEBUG
// progress probes written to mapped host memory (readable while the kernel runs):
// dbg[(cta * 4 + warp) * 32 + lane] = last recorded position of that thread
__device__ volatile int* g_nw_dbg;
#define NW_PROBE(v) (g_nw_dbg[(blockIdx.x * 4 + (threadIdx.x >> 5)) * 32 + (threadIdx.x & 31)] = (v))
// event times (globaltimer ns, low 32 bits): g_nw_trace[(cta * 4 + role) * 2048 + idx]
__device__ unsigned g_nw_trace[148 * 4 * 2048];
__device__ __forceinline__ unsigned nw_now() {
    unsigned t;
    asm volatile("mov.u32 %0, %%globaltimer_lo;" : "=r"(t));
    return t;
}
#define NW_TRACE(role, idx) \
    do { if ((idx) < 2048) g_nw_trace[(blockIdx.x * 4 + (role)) * 2048 + (idx)] = nw_now(); } while (0)
#else
#define NW_PROBE(v) ((void)0)
#define NW_TRACE(role, idx) ((void)0)
#endif

struct Ctrl {
    int strip;
    int loaded;      // sim blocks <= loaded have landed
    int computed;    // S' blocks <= computed are final
    int flushed;     // blocks <= flushed are written out (ring slot reusable)
    int ready;       // boundary rows < ready are in the shared ring
};

__device__ __forceinline__ int ldv(const int* p) { return *reinterpret_cast<const volatile int*>(p); }
__device__ __forceinline__ void stv(int* p, int v) { *reinterpret_cast<volatile int*>(p) = v; }

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async4(uint32_t dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" :: "r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" :: "n"(N) : "memory"); }

__device__ __forceinline__ int4 lds128(uint32_t a) {
    int4 v;
    asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
    return v;
}
// volatile: re-read on every spin iteration (ptxas hoists weak loads out of loops)
__device__ __forceinline__ int4 lds128v(uint32_t a) {
    int4 v;
    asm volatile("ld.volatile.shared.v4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts128(uint32_t a, int x, int y, int z, int w) {
    asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" :: "r"(a), "r"(x), "r"(y), "r"(z), "r"(w) : "memory");
}
__device__ __forceinline__ void sts64(uint32_t a, unsigned long long v) {
    asm volatile("st.shared.b64 [%0], %1;" :: "r"(a), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_tagged(const unsigned long long* p) {
    unsigned long long w;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(w) : "l"(p) : "memory");
    return w;
}
__device__ __forceinline__ void st_tagged(unsigned long long* p, unsigned long long w) {
    asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" :: "l"(p), "l"(w) : "memory");
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

// compute-warp state: S' of the lane's 4 columns in its last finished row,
// the diagonal predecessor of its first column, and the two values it sends
struct Lane {
    int h0, h1, h2, h3, dprev, vs3, ws3;
};

__device__ __forceinline__ int2 lds64v(uint32_t a) {
    int2 v;
    asm volatile("ld.volatile.shared.v2.b32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
    return v;
}

// predicated (branch-free) publication of two tagged boundary words
__device__ __forceinline__ void publish2(unsigned long long* p, int pred, int v0, unsigned t0, int v1, unsigned t1) {
    asm volatile(
        "{\n\t.reg .pred q;\n\t.reg .b64 a, b;\n\t"
        "setp.ne.s32 q, %1, 0;\n\t"
        "mov.b64 a, {%2, %3};\n\t"
        "mov.b64 b, {%4, %5};\n\t"
        "@q st.relaxed.gpu.global.v2.b64 [%0], {a, b};\n\t}"
        :: "l"(p), "r"(pred), "r"(v0), "r"(t0), "r"(v1), "r"(t1) : "memory");
}

// one anti-diagonal step of the compute warp: lane j computes the 2x4 block
// rows r0 = 2(s-j), r0+1, columns 4j..4j+3 of the strip
template <bool GUARD>
__device__ __forceinline__ void nw_step(Lane& c, int s, int lane, uint32_t ring_lane, uint32_t bnd, int p2,
                                        int n, unsigned long long* my_bnd, unsigned tagp1, int4& a_nx, int4& b_nx) {
    const int r0 = 2 * (s - lane);
    const uint32_t addr = ring_lane + (uint32_t)((r0 & (RING_ROWS - 1)) * ROW_BYTES);
    const int4 a = a_nx, b = b_nx;                      // sim rows r0, r0 + 1 (loaded one step ahead)
    {
        const uint32_t nx = ring_lane + (uint32_t)(((r0 + 2) & (RING_ROWS - 1)) * ROW_BYTES);
        a_nx = lds128(nx);
        b_nx = lds128(nx + ROW_BYTES);
    }
    // lane 0's left values: boundary rows 2s, 2s + 1 (readiness checked per 4 steps)
    const int2 bv = lds64v(bnd + (uint32_t)(((2 * s) & (RING_ROWS - 1)) * 4));
    // lane j-1 finished rows r0, r0 + 1 in the previous step
    const int sl0 = __shfl_up_sync(0xffffffffu, c.vs3, 1);
    const int sl1 = __shfl_up_sync(0xffffffffu, c.ws3, 1);
    const int left0 = lane == 0 ? bv.x : sl0;
    const int left1 = lane == 0 ? bv.y : sl1;
    // row r0 (up = h, diagonal = dprev / h), then row r0 + 1 (up = v)
    const int v0 = max(max(a.x + c.dprev + p2, c.h0), left0);
    const int v1 = max(max(a.y + c.h0 + p2, c.h1), v0);
    const int v2 = max(max(a.z + c.h1 + p2, c.h2), v1);
    const int v3 = max(max(a.w + c.h2 + p2, c.h3), v2);
    const int w0 = max(max(b.x + left0 + p2, v0), left1);
    const int w1 = max(max(b.y + v0 + p2, v1), w0);
    const int w2 = max(max(b.z + v1 + p2, v2), w1);
    const int w3 = max(max(b.w + v2 + p2, v3), w2);
    const bool live = !GUARD || r0 >= 0;                // lanes start one step apart
    if (live) {
        sts128(addr, v0, v1, v2, v3);                   // S' replaces sim in place
        sts128(addr + ROW_BYTES, w0, w1, w2, w3);
    }
    c.h0 = live ? w0 : c.h0;
    c.h1 = live ? w1 : c.h1;
    c.h2 = live ? w2 : c.h2;
    c.h3 = live ? w3 : c.h3;
    c.dprev = live ? left1 : c.dprev;
    c.vs3 = live ? v3 : c.vs3;
    c.ws3 = live ? w3 : c.ws3;
    // the strip's last column goes to the right neighbour (lane 31, rows < n)
    publish2(my_bnd + r0, (lane == 31) & (r0 < n) & live, v3, tagp1 + (unsigned)r0, w3, tagp1 + 1u + (unsigned)r0);
}

// 16 steps (32 rows of lane 0); boundary readiness is checked every 4 steps
// with a value prefetched 4 steps earlier
template <bool GUARD>
__device__ __forceinline__ void nw_block(Lane& c, int k, int lane, uint32_t ring_lane, uint32_t bnd, int p2, int n,
                                         unsigned long long* my_bnd, unsigned tagp1, int& rd, const int* ready,
                                         int4& a_nx, int4& b_nx) {
#pragma unroll
    for (int u = 0; u < STEPS; ++u) {
        if ((u & 3) == 0) {
            const int need = 2 * (k * STEPS + u) + 8;
            while (rd < need) rd = ldv(ready);
            rd = ldv(ready);
        }
        nw_step<GUARD>(c, k * STEPS + u, lane, ring_lane, bnd, p2, n, my_bnd, tagp1, a_nx, b_nx);
    }
}

__global__ void __launch_bounds__(128, 1)
nw_strips(const int32_t* __restrict__ sim, int32_t* __restrict__ score, int n, int p, int strips_per_matrix,
          int total_strips, int* __restrict__ ticket, unsigned long long* __restrict__ bnd_g, unsigned epoch) {
    extern __shared__ __align__(16) unsigned char smem[];
    int32_t* ring_gen = reinterpret_cast<int32_t*>(smem);
    Ctrl* ctrl = reinterpret_cast<Ctrl*>(smem + RING_BYTES + BND_BYTES);
    const uint32_t ring = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
    const uint32_t bnd = ring + RING_BYTES;
    const int lane = threadIdx.x & 31;
    const int warp = __shfl_sync(0xffffffffu, (int)threadIdx.x >> 5, 0);   // warp-uniform role
    const int n_pad = (n + BLK - 1) / BLK * BLK;
    const int nblocks = n_pad / BLK;
    const unsigned tag = (epoch & 0x7FFu) << 21;     // rows are < 2^20

    for (;;) {
        if (threadIdx.x == 0) {
            ctrl->strip = atomicAdd(ticket, 1);
            ctrl->loaded = ctrl->computed = ctrl->flushed = -1;
            ctrl->ready = 0;
        }
        __syncthreads();
        const int strip = ctrl->strip;
        NW_PROBE(6000000 + strip);
        if (strip >= total_strips) return;
        const int bm = strip / strips_per_matrix;
        const int w = strip - bm * strips_per_matrix;
        const int col0 = w * STRIP;
        unsigned long long* my_bnd = bnd_g + (long long)strip * n_pad;

        if (warp == 0) {
            // ---------------- compute ----------------
            Lane c = {0, 0, 0, 0, 0, 0, 0};
            const int p2 = 2 * p;
            const uint32_t ring_lane = ring + 16u * lane;
            const unsigned tagp1 = tag + 1u;
            int pl = ldv(&ctrl->loaded);
            int rd = ldv(&ctrl->ready);
            int4 a_nx = make_int4(0, 0, 0, 0), b_nx = make_int4(0, 0, 0, 0);
            for (int k = 0; k < nblocks + DRAIN; ++k) {
                NW_PROBE(1000000 + k);
                if (lane == 0) NW_TRACE(0, k);
                if (k >= 3) {                           // lane 31 finished block k-3 at step 16k-2
                    __syncwarp();
                    if (lane == 0) stv(&ctrl->computed, k - 3);
                }
                // the last step of block k prefetches block k+1's first rows: need both
                const int need_blk = min(k + 1, nblocks + DRAIN - 1);
                while (pl < need_blk) pl = ldv(&ctrl->loaded);
                if (k == 0) {                           // first step's operands
                    const uint32_t a0 = ring_lane + (uint32_t)(((-2 * lane) & (RING_ROWS - 1)) * ROW_BYTES);
                    a_nx = lds128(a0);
                    b_nx = lds128(a0 + ROW_BYTES);
                }
                pl = ldv(&ctrl->loaded);                // prefetch for the next block
                if (k < 2)
                    nw_block<true>(c, k, lane, ring_lane, bnd, p2, n, my_bnd, tagp1, rd, &ctrl->ready, a_nx, b_nx);
                else
                    nw_block<false>(c, k, lane, ring_lane, bnd, p2, n, my_bnd, tagp1, rd, &ctrl->ready, a_nx, b_nx);
            }
            __syncwarp();
            if (lane == 0) stv(&ctrl->computed, nblocks + DRAIN - 1);
        } else if (warp == 1) {
            // ---------------- producer: sim blocks -> ring ----------------
            const int32_t* simb = sim + (long long)bm * n * n;
            const bool vec = (n & 3) == 0;
            for (int k = 0; k < nblocks + DRAIN; ++k) {
                NW_PROBE(2000000 + k);
                if (k >= NSLOT) {
                    while (ldv(&ctrl->flushed) < k - NSLOT) __nanosleep(128);
                }
                if (k < nblocks) {
                    const int rows = min(BLK, n - k * BLK);
                    uint32_t dst = ring + (uint32_t)((k & (NSLOT - 1)) * BLK * ROW_BYTES);
                    if (vec) {
                        const bool ok = col0 + CPL * lane < n;
                        const int32_t* src = simb + (long long)k * BLK * n + col0 + CPL * lane;
                        dst += 16u * lane;
#pragma unroll 8
                        for (int r = 0; r < rows; ++r) {
                            if (ok) cp_async16(dst, src);
                            dst += ROW_BYTES;
                            src += n;
                        }
                    } else {
                        const int32_t* src = simb + (long long)k * BLK * n + col0 + lane;
                        dst += 4u * lane;
                        for (int r = 0; r < rows; ++r) {
#pragma unroll
                            for (int q = 0; q < CPL; ++q)
                                if (col0 + 32 * q + lane < n) cp_async4(dst + 128u * q, src + 32 * q);
                            dst += ROW_BYTES;
                            src += n;
                        }
                    }
                }
                cp_async_commit();
                if (k >= 2) {
                    cp_async_wait<2>();
                    __syncwarp();
                    if (lane == 0) { stv(&ctrl->loaded, k - 2); NW_TRACE(1, k - 2); }
                }
            }
            cp_async_wait<0>();
            __syncwarp();
            if (lane == 0) stv(&ctrl->loaded, nblocks + DRAIN - 1);
        } else if (warp == 2) {
            // ---------------- boundary: left strip's last column -> shared ring ----------------
            // Lane l polls row 32m + l; rows are handed to the compute warp in
            // order through ctrl->ready as soon as a prefix of the group is in.
            const unsigned long long* left = my_bnd - n_pad;
            const int groups = nblocks + DRAIN;
            for (int m = 0; m < groups; ++m) {
                const int r = m * BLK + lane;
                NW_PROBE(3000000 + r);
                if (m >= NSLOT) {
                    while (ldv(&ctrl->computed) < m - NSLOT) __nanosleep(128);
                }
                int v = 0;                              // S'[r+1][0] = 0 on the matrix edge
                bool ok = true;
                if (w > 0 && r < n) {
                    const unsigned long long x = ld_tagged(left + r);
                    ok = (unsigned)(x >> 32) == (tag | (unsigned)(r + 1));
                    v = (int)(unsigned)x;
                }
                bool written = false;
                int told = 0;
                for (;;) {
                    const unsigned ball = __ballot_sync(0xffffffffu, ok);
                    const int t = ball == 0xffffffffu ? 32 : __ffs(~ball) - 1;   // ready prefix
                    if (ok && !written && lane < t) {
                        asm volatile("st.shared.b32 [%0], %1;" :: "r"(bnd + (uint32_t)((r & (RING_ROWS - 1)) * 4)),
                                     "r"(v) : "memory");
                        written = true;
                    }
                    if (t > told) {
                        __syncwarp();
                        if (lane == 0) stv(&ctrl->ready, m * BLK + t);
                        told = t;
                    }
                    if (t == 32) break;
                    __nanosleep(NW_POLL_NS);
                    if (!ok) {
                        const unsigned long long x = ld_tagged(left + r);
                        ok = (unsigned)(x >> 32) == (tag | (unsigned)(r + 1));
                        v = (int)(unsigned)x;
                    }
                }
                if (lane == 31) NW_TRACE(2, m);
            }
        } else {
            // ---------------- flusher: S' -> S, coalesced row segments ----------------
            int32_t* sc = score + (long long)bm * ((long long)n + 1) * ((long long)n + 1);
            const long long ld = (long long)n + 1;
            bool ok[CPL];
#pragma unroll
            for (int q = 0; q < CPL; ++q) ok[q] = col0 + 32 * q + lane < n;
            for (int k = 0; k < nblocks; ++k) {
                NW_PROBE(5000000 + k);
                while (ldv(&ctrl->computed) < k) __nanosleep(64);
                const int rows = min(BLK, n - k * BLK);
                const int32_t* src = ring_gen + (k & (NSLOT - 1)) * BLK * STRIP + lane;
                int32_t* dst = sc + (long long)(k * BLK + 1) * ld + col0 + 1 + lane;
                int off = (k * BLK + col0 + lane + 2) * p;     // (i + j) * p of column lane, row k*BLK
#pragma unroll 4
                for (int r = 0; r < rows; ++r) {
#pragma unroll
                    for (int q = 0; q < CPL; ++q)
                        if (ok[q]) dst[32 * q] = src[32 * q] - (off + 32 * q * p);
                    dst += ld;
                    src += STRIP;
                    off += p;
                }
                __syncwarp();
                if (lane == 0) { stv(&ctrl->flushed, k); NW_TRACE(3, k); }
            }
        }
        __syncthreads();
    }
}

}  // namespace

#ifdef LEGO_NW_DEBUG
static int* lego_nw_dbg_host = nullptr;
static void* g_nw_trace_ptr() {
    void* p = nullptr;
    cudaGetSymbolAddress(&p, g_nw_trace);
    return p;
}
// snapshot of the progress probes (debug builds only)
extern "C" int lego_nw_debug_trace(unsigned* out) {
    return cudaMemcpyFromSymbol(out, g_nw_trace, sizeof(g_nw_trace)) == cudaSuccess ? 148 * 4 * 2048 : 0;
}
extern "C" int lego_nw_debug_snapshot(int* out, int count) {
    if (!lego_nw_dbg_host) return 0;
    const int m = count < 148 * 4 * 32 ? count : 148 * 4 * 32;
    for (int i = 0; i < m; ++i) out[i] = ((volatile int*)lego_nw_dbg_host)[i];
    return m;
}
#endif

// Boundary words + tickets, kept per (device, stream) across calls: words are
// tagged with a launch epoch, so a launch never mistakes a previous launch's
// word for its own; tickets are one counter per epoch.  The buffer is zeroed
// when it is (re)allocated and whenever the 11-bit epoch wraps.  Launches on
// one stream are ordered, so sharing the buffer between them is safe.
struct NwScratch {
    char* buf = nullptr;
    size_t bytes = 0;
    unsigned epoch = 0;
};
constexpr size_t NW_TICKETS = 2048 * sizeof(int);

static lego_status nw_scratch(cudaStream_t st, size_t bnd_bytes, int** ticket, unsigned long long** bnd,
                              unsigned* epoch) {
    static std::mutex mu;
    static std::map<std::pair<int, cudaStream_t>, NwScratch> cache;
    int dev = 0;
    LEGO_TRY(lego_cuda_check(cudaGetDevice(&dev), "cudaGetDevice"));
    std::lock_guard<std::mutex> lk(mu);
    NwScratch& e = cache[std::make_pair(dev, st)];
    const size_t need = NW_TICKETS + bnd_bytes;
    bool zero = false;
    if (e.bytes < need) {
        if (e.buf) LEGO_TRY(lego_cuda_check(cudaFreeAsync(e.buf, st), "cudaFreeAsync"));
        e.buf = nullptr;
        e.bytes = 0;
        const size_t grow = need + need / 4;
        LEGO_TRY(lego_cuda_check(cudaMallocAsync((void**)&e.buf, grow, st), "cudaMallocAsync"));
        e.bytes = grow;
        zero = true;
    }
    e.epoch = (e.epoch + 1) & 0x7FFu;
    if (e.epoch == 0) {
        e.epoch = 1;
        zero = true;
    }
    if (zero) {
        LEGO_TRY(lego_cuda_check(cudaMemsetAsync(e.buf, 0, e.bytes, st), "cudaMemsetAsync"));
        e.epoch = 1;
    }
    *ticket = reinterpret_cast<int*>(e.buf) + e.epoch;
    *bnd = reinterpret_cast<unsigned long long*>(e.buf + NW_TICKETS);
    *epoch = e.epoch;
    return LEGO_OK;
}

extern "C" lego_status lego_nw_i32(const int32_t* sim, int32_t* score, int64_t n, int32_t penalty, int64_t batch,
                                   void* stream) {
    if (n < 0 || batch < 0) return lego_fail(LEGO_E_SHAPE, "negative NW size");
    if (batch == 0) return LEGO_OK;
    if (n > (1 << 20)) return lego_fail(LEGO_E_SHAPE, "NW n above 2^20");
    if (!sim || !score) return lego_fail(LEGO_E_ARG, "null buffer");
    if ((uintptr_t)sim & 15) return lego_fail(LEGO_E_ARG, "sim must be 16-byte aligned");
    if ((long long)std::llabs((long long)penalty) * (2 * n + 2) >= (1LL << 30))
        return lego_fail(LEGO_E_ARG, "|penalty| * (2n + 2) must stay below 2^30 (offset scores are int32)");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const long long w = n + 1;
    const long long bgrid = (batch * w + 255) / 256;
    nw_borders<<<(unsigned)(bgrid < 4096 ? bgrid : 4096), 256, 0, st>>>(score, n, penalty, batch);
    if (n == 0) return lego_cuda_check(cudaGetLastError(), "nw borders");
    const int strips = (int)((n + STRIP - 1) / STRIP);
    const long long total = (long long)strips * batch;
    if (total > INT32_MAX) return lego_fail(LEGO_E_SHAPE, "NW batch too large");
    const long long n_pad = (n + BLK - 1) / BLK * BLK;
    const size_t bnd_bytes = sizeof(unsigned long long) * (size_t)total * (size_t)n_pad;
    int* ticket = nullptr;
    unsigned long long* bnd_g = nullptr;
    unsigned epoch = 0;
    LEGO_TRY(nw_scratch(st, bnd_bytes, &ticket, &bnd_g, &epoch));
    static cudaError_t attr = cudaFuncSetAttribute(nw_strips, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   SMEM_BYTES);
    LEGO_TRY(lego_cuda_check(attr, "cudaFuncSetAttribute(nw)"));
#ifdef LEGO_NW_DEBUG
    static int* host_dbg = nullptr;
    if (!host_dbg) {
        cudaHostAlloc((void**)&host_dbg, 148 * 4 * 32 * sizeof(int), cudaHostAllocMapped);
        int* dptr = nullptr;
        cudaHostGetDevicePointer((void**)&dptr, host_dbg, 0);
        cudaMemcpyToSymbol(g_nw_dbg, &dptr, sizeof(dptr));
        lego_nw_dbg_host = host_dbg;
    }
    memset(host_dbg, 0xff, 148 * 4 * 32 * sizeof(int));
    cudaMemsetAsync(g_nw_trace_ptr(), 0, 148 * 4 * 2048 * sizeof(unsigned), st);
#endif
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const long long ctas = total < sms ? total : sms;      // one strip CTA per SM, persistent
    nw_strips<<<(unsigned)ctas, 128, SMEM_BYTES, st>>>(sim, score, (int)n, penalty, strips, (int)total, ticket,
                                                       bnd_g, epoch);
    return lego_cuda_check(cudaGetLastError(), "nw launch");
}
