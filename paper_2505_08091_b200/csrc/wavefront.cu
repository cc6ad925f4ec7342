// wavefront.cu -- Needleman-Wunsch anti-diagonal wavefront (config 4b).
// (first version: placeholder until the tiled kernel lands)
#include "lego_common.h"

extern "C" lego_status lego_nw_i32(const int32_t* sim, int32_t* score, int64_t n, int32_t penalty,
                                   int64_t batch, void* stream) {
    (void)sim; (void)score; (void)n; (void)penalty; (void)batch; (void)stream;
    return lego_fail(LEGO_E_UNSUPPORTED, "lego_nw_i32 not built yet");
}
