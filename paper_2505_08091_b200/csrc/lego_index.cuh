// lego_index.cuh -- device helpers for generated LEGO index code (sm_100a).
//
// Semantics follow the reference Expr evaluator (pkg/src/lego/expr.py:261-298):
// floor division, Python-sign modulo (result has the divisor's sign), exact
// integer square root.  Self-contained (no std headers) so NVRTC can compile
// it without a CUDA include path.
#pragma once

typedef unsigned long long lego_u64;
typedef long long lego_i64;

static __device__ __forceinline__ long long lego_fdiv(long long a, long long b) {
    if (b == 0) return 0;                       // unreachable for valid layouts
    long long q = a / b;
    return (a % b != 0 && ((a < 0) != (b < 0))) ? q - 1 : q;
}
static __device__ __forceinline__ int lego_fdiv(int a, int b) {
    if (b == 0) return 0;
    int q = a / b;
    return (a % b != 0 && ((a < 0) != (b < 0))) ? q - 1 : q;
}
static __device__ __forceinline__ long long lego_fmod(long long a, long long b) {
    if (b == 0) return 0;
    long long r = a % b;
    return (r != 0 && ((r < 0) != (b < 0))) ? r + b : r;
}
static __device__ __forceinline__ int lego_fmod(int a, int b) {
    if (b == 0) return 0;
    int r = a % b;
    return (r != 0 && ((r < 0) != (b < 0))) ? r + b : r;
}

// exact floor(sqrt(x)); negative arguments clamp to 0 (only reachable in the
// untaken arm of a select, which the generated code evaluates eagerly)
static __device__ __forceinline__ int lego_isqrt32(int x) {
    if (x <= 0) return 0;
    int r = (int)sqrtf((float)x);
    while ((long long)r * r > x) --r;
    while ((long long)(r + 1) * (r + 1) <= x) ++r;
    return r;
}
static __device__ __forceinline__ long long lego_isqrt64(long long x) {
    if (x <= 0) return 0;
    long long r = (long long)sqrt((double)x);
    while (r * r > x) --r;
    while ((r + 1) * (r + 1) <= x) ++r;
    return r;
}
