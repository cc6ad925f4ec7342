// lego_common.h -- shared host-side helpers of liblego_b200.so.
#pragma once
#include <cuda_runtime.h>

#include <atomic>

#include "../../include/lego_b200.h"

// record a failure (thread-local message) and return its code
lego_status lego_fail(lego_status code, const char* fmt, ...);
lego_status lego_cuda_check(cudaError_t e, const char* what);

#define LEGO_TRY(expr)                      \
    do {                                    \
        lego_status _s = (expr);            \
        if (_s != LEGO_OK) return _s;       \
    } while (0)

// Needleman-Wunsch launch plan (wavefront.cu): validated sizes, tile grid and
// the per-(device, stream) scratch, preset for one launch on `st`.
struct NwPlan {
    long long n, batch;
    int H, nr, nc, total;     // tile rows, tile grid, tickets (batch * nr * nc)
    int* ticket;              // claim counter (zeroed)
    int* bnd;                 // right-column words per (matrix, tile column) (NW_EMPTY)
    int* top;                 // tiled: bottom-row words per (matrix, tile) (NW_EMPTY), else null
    unsigned ctas, border_ctas;
    int smem;
};
lego_status lego_nw_prepare(const int32_t* sim, int32_t* score, int64_t n, int32_t penalty, int64_t batch,
                            int64_t tile_rows, int tiled, cudaStream_t st, NwPlan* plan);
int lego_nw_smem_bytes();   // dynamic shared memory of the wavefront kernel (nw_kernels.cuh)

// The >48 KiB dynamic shared memory opt-in is a per-device function
// attribute: set it once per device (bit d of `done`) before launching.
template <typename Kernel>
static inline lego_status lego_smem_optin(Kernel kernel, int bytes, std::atomic<unsigned long long>& done,
                                          const char* what) {
    int dev = 0;
    LEGO_TRY(lego_cuda_check(cudaGetDevice(&dev), "cudaGetDevice"));
    const unsigned long long bit = 1ull << (dev & 63);
    if (done.load() & bit) return LEGO_OK;
    LEGO_TRY(lego_cuda_check(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes),
                             what));
    done.fetch_or(bit);
    return LEGO_OK;
}
