// lego_common.h -- shared host-side helpers of liblego_b200.so.
#pragma once
#include <cuda_runtime.h>

#include "../../include/lego_b200.h"

// record a failure (thread-local message) and return its code
lego_status lego_fail(lego_status code, const char* fmt, ...);
lego_status lego_cuda_check(cudaError_t e, const char* what);

#define LEGO_TRY(expr)                      \
    do {                                    \
        lego_status _s = (expr);            \
        if (_s != LEGO_OK) return _s;       \
    } while (0)
