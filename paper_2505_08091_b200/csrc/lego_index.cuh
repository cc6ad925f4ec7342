// lego_index.cuh -- device helpers for generated LEGO index code (sm_100a).
//
// Semantics follow the reference Expr evaluator (pkg/src/lego/expr.py:261-298):
// floor division, Python-sign modulo (result has the divisor's sign), exact
// integer square root.  Self-contained (no std headers) so NVRTC can compile
// it without a CUDA include path.  The division helpers are templates so a
// 64-bit numerator with a 32-bit literal divisor (what emit.CUDA_PROFILE
// prints) computes in the wider type.
#pragma once

typedef unsigned long long lego_u64;
typedef long long lego_i64;

template <typename A, typename B>
static __device__ __forceinline__ auto lego_fdiv(A a, B b) -> decltype(a + b) {
    typedef decltype(a + b) T;
    const T x = (T)a, y = (T)b;
    if (y == 0) return 0;                       // unreachable for valid layouts
    const T q = x / y;
    return (x % y != 0 && ((x < 0) != (y < 0))) ? q - 1 : q;
}
template <typename A, typename B>
static __device__ __forceinline__ auto lego_fmod(A a, B b) -> decltype(a + b) {
    typedef decltype(a + b) T;
    const T x = (T)a, y = (T)b;
    if (y == 0) return 0;
    const T r = x % y;
    return (r != 0 && ((r < 0) != (y < 0))) ? r + y : r;
}

// exact floor(sqrt(x)); negative arguments clamp to 0 (only reachable in the
// untaken arm of a select, which the generated code evaluates eagerly)
// 32-bit: x < 2^31, so float(x) (rel. error 2^-24) and the approximate
// MUFU square root (rel. error ~2^-22) land within 0.02 of sqrt(x) <= 46341;
// the truncated root is off by at most one and one branch-free correction
// step each way is exact
// branch-free: the clamp is a max, and .ftz drops the denormal rescaling
// (float(x) >= 1 or 0); checked exhaustively over [0, 2^31) and a sample of
// negative arguments by scripts/micro/isqrt_exhaustive.cu
static __device__ __forceinline__ int lego_isqrt32(int x) {
    const unsigned ux = (unsigned)max(x, 0);
    float fr;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(fr) : "f"((float)ux));
    unsigned r = (unsigned)fr;
    r -= (r * r > ux) ? 1u : 0u;
    r += ((r + 1u) * (r + 1u) <= ux) ? 1u : 0u;
    return (int)r;
}
static __device__ __forceinline__ long long lego_isqrt64(long long x) {
    if (x <= 0) return 0;
    long long r = (long long)sqrt((double)x);
    while (r * r > x) --r;
    while ((r + 1) * (r + 1) <= x) ++r;
    return r;
}
// overloads used by the `cuda` emit profile (emit.CUDA_PROFILE, template splices)
static __device__ __forceinline__ int lego_isqrt(int x) { return lego_isqrt32(x); }
static __device__ __forceinline__ long long lego_isqrt(long long x) { return lego_isqrt64(x); }
