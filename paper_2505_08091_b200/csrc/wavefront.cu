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

lego_status lego_nw_prepare(const int32_t* sim, int32_t* score, int64_t n, int32_t penalty, int64_t batch,
                            int64_t tile_rows, int tiled, cudaStream_t st, NwPlan* plan) {
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
    if (n == 0) return LEGO_OK;
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
