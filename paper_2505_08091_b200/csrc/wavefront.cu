// wavefront.cu -- host side of the Needleman-Wunsch wavefront (BASELINE.json
// config 4b) and the library's built-in instance of the kernel template
// (nw_kernels.cuh) for the default layout: column strips of 128 columns
// (tile order row-major over a 1 x ceil(n/128) tile grid, row-major ring).
// Programs generated from other LEGO layouts (kernels.nw_program) are
// compiled from the same template by NVRTC and launched through
// lego_nw_run (lego_runtime.cu), sharing lego_nw_prepare below.
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <utility>

#include "lego_common.h"

#define NW_GLOBAL static __global__
#define NW_BAND_ENTRY 1
#include "nw_kernels.cuh"

#ifdef LEGO_NW_DEBUG
// snapshot of the per-role event times (debug builds only)
extern "C" int lego_nw_debug_trace(unsigned* out) {
    return cudaMemcpyFromSymbol(out, nwk::g_nw_trace, sizeof(nwk::g_nw_trace)) == cudaSuccess ? 148 * 4 * 2048 : 0;
}
#endif

// Boundary words + ticket, kept per (device, stream) across calls (launches
// on one stream are ordered, so they can share it); every launch presets the
// words it uses to NW_EMPTY and the ticket to 0.
struct NwScratch {
    char* buf = nullptr;
    size_t bytes = 0;
};
constexpr size_t NW_TICKET_BYTES = 256;

static lego_status nw_scratch(cudaStream_t st, size_t words_bytes, int** ticket, int** words) {
    static std::mutex mu;
    static std::map<std::pair<int, cudaStream_t>, NwScratch> cache;
    int dev = 0;
    LEGO_TRY(lego_cuda_check(cudaGetDevice(&dev), "cudaGetDevice"));
    std::lock_guard<std::mutex> lk(mu);
    NwScratch& e = cache[std::make_pair(dev, st)];
    const size_t need = NW_TICKET_BYTES + words_bytes;
    if (e.bytes < need) {
        if (e.buf) LEGO_TRY(lego_cuda_check(cudaFreeAsync(e.buf, st), "cudaFreeAsync"));
        e.buf = nullptr;
        e.bytes = 0;
        const size_t grow = need + need / 4;
        LEGO_TRY(lego_cuda_check(cudaMallocAsync((void**)&e.buf, grow, st), "cudaMallocAsync"));
        e.bytes = grow;
    }
    LEGO_TRY(lego_cuda_check(cudaMemsetAsync(e.buf, 0, NW_TICKET_BYTES, st), "cudaMemsetAsync"));
    if (words_bytes)
        LEGO_TRY(lego_cuda_check(cudaMemsetAsync(e.buf + NW_TICKET_BYTES, 0x80, words_bytes, st),
                                 "cudaMemsetAsync"));
    *ticket = reinterpret_cast<int*>(e.buf);
    *words = reinterpret_cast<int*>(e.buf + NW_TICKET_BYTES);
    return LEGO_OK;
}

int lego_nw_smem_bytes() { return nwk::SMEM_BYTES; }

// argument rules shared by every NW entry point; fills the border grid
static lego_status nw_validate(const int32_t* sim, int32_t* score, int64_t n, int32_t penalty, int64_t batch,
                               NwPlan* plan) {
    memset(plan, 0, sizeof *plan);
    if (n < 0 || batch < 0) return lego_fail(LEGO_E_SHAPE, "negative NW size");
    if (n > (1 << 20)) return lego_fail(LEGO_E_SHAPE, "NW n above 2^20");
    if (batch == 0) return LEGO_OK;
    if (!score || (n > 0 && !sim)) return lego_fail(LEGO_E_ARG, "null buffer");
    if ((uintptr_t)sim & 15) return lego_fail(LEGO_E_ARG, "sim must be 16-byte aligned");
    if ((uintptr_t)score & 3) return lego_fail(LEGO_E_ARG, "score must be 4-byte aligned");
    if ((long long)std::llabs((long long)penalty) * (2 * n + 2) >= (1LL << 30))
        return lego_fail(LEGO_E_ARG, "|penalty| * (2n + 2) must stay below 2^30 (offset scores are int32)");
    plan->n = n;
    plan->batch = batch;
    const long long bgrid = (batch * (n + 1) + 255) / 256;
    plan->border_ctas = (unsigned)(bgrid < 4096 ? bgrid : 4096);
    return LEGO_OK;
}

lego_status lego_nw_prepare(const int32_t* sim, int32_t* score, int64_t n, int32_t penalty, int64_t batch,
                            int64_t tile_rows, int tiled, cudaStream_t st, NwPlan* plan) {
    LEGO_TRY(nw_validate(sim, score, n, penalty, batch, plan));
    if (batch == 0 || n == 0) return LEGO_OK;
    const long long H = tile_rows > 0 ? tile_rows : n;
    const long long nr = (n + H - 1) / H;
    const long long nc = (n + nwk::STRIP - 1) / nwk::STRIP;
    if (nr > 1 && (H % nwk::BLK)) return lego_fail(LEGO_E_SHAPE, "tile rows must be a multiple of 32");
    if (nr > 1 && !tiled) return lego_fail(LEGO_E_ARG, "a strip program cannot run tiles of %lld rows", H);
    const long long total = nr * nc * batch;
    if (total > INT32_MAX / 2) return lego_fail(LEGO_E_SHAPE, "NW batch too large");
    const long long n_pad = (n + nwk::BLK - 1) / nwk::BLK * nwk::BLK;
    const size_t bnd_words = (size_t)(nc * batch) * (size_t)n_pad;
    const size_t top_words = tiled ? (size_t)total * nwk::STRIP : 0;
    int* ticket = nullptr;
    int* words = nullptr;
    LEGO_TRY(nw_scratch(st, sizeof(int) * (bnd_words + top_words), &ticket, &words));
    int dev = 0, sms = 148;
    LEGO_TRY(lego_cuda_check(cudaGetDevice(&dev), "cudaGetDevice"));
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    plan->H = (int)H;
    plan->nr = (int)nr;
    plan->nc = (int)nc;
    plan->total = (int)total;
    plan->ticket = ticket;
    plan->bnd = words;
    plan->top = tiled ? words + bnd_words : nullptr;
    plan->ctas = (unsigned)(total < sms ? total : sms);     // one CTA per SM, persistent
    plan->smem = nwk::SMEM_BYTES;
    return LEGO_OK;
}

extern "C" lego_status lego_nw_i32(const int32_t* sim, int32_t* score, int64_t n, int32_t penalty, int64_t batch,
                                   void* stream) {
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    NwPlan pl;
    LEGO_TRY(lego_nw_prepare(sim, score, n, penalty, batch, n, 0, st, &pl));
    if (batch == 0) return LEGO_OK;
    lego_nw_borders<<<pl.border_ctas, 256, 0, st>>>(score, n, penalty, batch);
    if (n == 0) return lego_cuda_check(cudaGetLastError(), "nw borders");
    static std::atomic<unsigned long long> attr_set{0};
    LEGO_TRY(lego_smem_optin(lego_nw_tiles, nwk::SMEM_BYTES, attr_set, "cudaFuncSetAttribute(nw)"));
#ifdef LEGO_NW_DEBUG
    {
        void* trace = nullptr;
        cudaGetSymbolAddress(&trace, nwk::g_nw_trace);
        cudaMemsetAsync(trace, 0, sizeof(nwk::g_nw_trace), st);
    }
#endif
    lego_nw_tiles<<<pl.ctas, 128, pl.smem, st>>>(sim, score, (int)n, penalty, pl.H, pl.nr, pl.nc, pl.total,
                                                  pl.ticket, pl.bnd, pl.top);
    return lego_cuda_check(cudaGetLastError(), "nw launch");
}

// Column band of a strip-mode NW (multi-GPU single alignment: shard.nw_score_banded).
// This launch computes strips [strip_begin, strip_end) of every matrix into the
// full-size score; bnd_words holds those strips' right-edge columns (batch x
// strips x n_pad int32, n_pad = n rounded up to 32), preset by the caller to
// the 0x80808080 sentinel before any reader starts; left_words is the previous
// band's last edge column (matrix b at left_words + b * left_batch_stride),
// possibly a peer GPU's memory, or null when strip_begin == 0.  Edges are
// published and polled at system scope.  max_ctas > 0 caps the persistent
// grid (several bands sharing one GPU must all be resident).
extern "C" lego_status lego_nw_band_i32(const int32_t* sim, int32_t* score, int64_t n, int32_t penalty,
                                        int64_t batch, int64_t strip_begin, int64_t strip_end, int32_t* bnd_words,
                                        const int32_t* left_words, int64_t left_batch_stride, int32_t max_ctas,
                                        void* stream) {
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (n < 1 || batch < 0) return lego_fail(LEGO_E_SHAPE, "NW band needs n >= 1");
    const long long nc = (n + nwk::STRIP - 1) / nwk::STRIP;
    if (strip_begin < 0 || strip_end > nc || strip_begin >= strip_end)
        return lego_fail(LEGO_E_SHAPE, "strip band [%lld, %lld) outside [0, %lld)", (long long)strip_begin,
                         (long long)strip_end, nc);
    if (!bnd_words || ((uintptr_t)bnd_words & 15)) return lego_fail(LEGO_E_ARG, "bnd_words must be 16-byte aligned");
    if ((strip_begin > 0) != (left_words != nullptr))
        return lego_fail(LEGO_E_ARG, "left_words is required exactly when the band does not start at strip 0");
    const long long n_pad = (n + nwk::BLK - 1) / nwk::BLK * nwk::BLK;
    if (left_words && left_batch_stride < n_pad) return lego_fail(LEGO_E_ARG, "left_batch_stride below n_pad");
    NwPlan pl;
    LEGO_TRY(nw_validate(sim, score, n, penalty, batch, &pl));   // the edge words are the caller's
    if (batch == 0) return LEGO_OK;
    int* ticket = nullptr;
    int* unused = nullptr;
    LEGO_TRY(nw_scratch(st, 0, &ticket, &unused));
    const long long nb = strip_end - strip_begin;
    const long long total = nb * batch;
    if (total > INT32_MAX / 2) return lego_fail(LEGO_E_SHAPE, "NW band batch too large");
    int dev = 0, sms = 148;
    LEGO_TRY(lego_cuda_check(cudaGetDevice(&dev), "cudaGetDevice"));
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    long long ctas = total < sms ? total : sms;
    if (max_ctas > 0 && ctas > max_ctas) ctas = max_ctas;
    lego_nw_borders<<<pl.border_ctas, 256, 0, st>>>(score, n, penalty, batch);
    static std::atomic<unsigned long long> attr_set{0};
    LEGO_TRY(lego_smem_optin(lego_nw_band, nwk::SMEM_BYTES, attr_set, "cudaFuncSetAttribute(nw band)"));
    lego_nw_band<<<(unsigned)ctas, 128, nwk::SMEM_BYTES, st>>>(sim, score, (int)n, penalty, (int)nc, (int)total,
                                                               ticket, bnd_words, (int)strip_begin, (int)nb,
                                                               left_words, (long long)left_batch_stride);
    return lego_cuda_check(cudaGetLastError(), "nw band launch");
}
