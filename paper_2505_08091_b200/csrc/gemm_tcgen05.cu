// gemm_tcgen05.cu -- bf16 GEMM on tcgen05/TMEM (config 5).
// (first version: placeholder until the tcgen05 kernel lands)
#include "lego_common.h"

extern "C" lego_status lego_gemm_bf16(const void* A, const void* B, void* C, int64_t M, int64_t N,
                                      int64_t K, int64_t batch, int32_t raster, void* stream) {
    (void)A; (void)B; (void)C; (void)M; (void)N; (void)K; (void)batch; (void)raster; (void)stream;
    return lego_fail(LEGO_E_UNSUPPORTED, "lego_gemm_bf16 not built yet");
}
