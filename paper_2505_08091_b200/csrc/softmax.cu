// softmax.cu -- row softmax, fp32, one CTA per row (BASELINE.json config 3).
//
// Thread/data layout is the LEGO layout
//     GroupBy([rows], [cols/(4T)], [T], [4]).OrderBy(Row(rows, cols))
// i.e. element (row, it, tid, v) lives at row*cols + it*4T + tid*4 + v
// (tests/test_softmax_layout.py derives this offset with apply_symbolic):
// every warp access is a coalesced float4, and a row is held in registers,
// so HBM sees one read and one write per element.  When a row does not fit
// the register budget the kernel streams it twice (online max/sum, then the
// normalised write).
#include <cuda_runtime.h>

#include "lego_common.h"

namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// block-wide reduction through shared memory (8 warps)
template <bool IsMax>
__device__ __forceinline__ float block_reduce(float v, float* red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    v = IsMax ? warp_max(v) : warp_sum(v);
    if (lane == 0) red[warp] = v;
    __syncthreads();
    float r = lane < (kThreads / 32) ? red[lane] : (IsMax ? -INFINITY : 0.f);
    r = IsMax ? warp_max(r) : warp_sum(r);
    __syncthreads();
    return r;
}

__device__ __forceinline__ float4 ld_stream(const float4* p) {
    float4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
    return v;
}
__device__ __forceinline__ void st_stream(float4* p, float4 v) {
    asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" :: "l"(p), "f"(v.x), "f"(v.y), "f"(v.z),
                 "f"(v.w) : "memory");
}

constexpr float kLog2e = 1.4426950408889634f;

// IT = float4 vectors per thread: the whole row lives in registers
template <int IT>
__global__ void __launch_bounds__(kThreads) softmax_rows_reg(const float* __restrict__ x,
                                                             float* __restrict__ y, long long cols) {
    __shared__ float red[kThreads / 32];
    const long long row = blockIdx.x;
    const float4* xr = reinterpret_cast<const float4*>(x + row * cols);
    float4* yr = reinterpret_cast<float4*>(y + row * cols);
    const int nvec = (int)(cols >> 2);
    float4 v[IT];
    float m = -INFINITY;
#pragma unroll
    for (int it = 0; it < IT; ++it) {
        const int k = it * kThreads + threadIdx.x;          // offset it*4T + tid*4 (in floats)
        v[it] = k < nvec ? ld_stream(xr + k) : make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
        m = fmaxf(m, fmaxf(fmaxf(v[it].x, v[it].y), fmaxf(v[it].z, v[it].w)));
    }
    m = block_reduce<true>(m, red);
    const float mb = m * kLog2e;
    float s = 0.f;
#pragma unroll
    for (int it = 0; it < IT; ++it) {
        v[it].x = exp2f(fmaf(v[it].x, kLog2e, -mb));
        v[it].y = exp2f(fmaf(v[it].y, kLog2e, -mb));
        v[it].z = exp2f(fmaf(v[it].z, kLog2e, -mb));
        v[it].w = exp2f(fmaf(v[it].w, kLog2e, -mb));
        s += (v[it].x + v[it].y) + (v[it].z + v[it].w);
    }
    s = block_reduce<false>(s, red);
    const float inv = 1.f / s;
#pragma unroll
    for (int it = 0; it < IT; ++it) {
        const int k = it * kThreads + threadIdx.x;
        if (k < nvec)
            st_stream(yr + k, make_float4(v[it].x * inv, v[it].y * inv, v[it].z * inv, v[it].w * inv));
    }
}

// long rows: online (max, sum) pass, then a normalising pass
__global__ void __launch_bounds__(kThreads) softmax_rows_stream(const float* __restrict__ x,
                                                                float* __restrict__ y, long long cols) {
    __shared__ float red[kThreads / 32];
    const long long row = blockIdx.x;
    const float4* xr = reinterpret_cast<const float4*>(x + row * cols);
    float4* yr = reinterpret_cast<float4*>(y + row * cols);
    const long long nvec = cols >> 2;
    float m = -INFINITY, s = 0.f;
    for (long long k = threadIdx.x; k < nvec; k += kThreads) {
        float4 v = xr[k];
        float mv = fmaxf(fmaxf(v.x, v.y), fmaxf(v.z, v.w));
        float nm = fmaxf(m, mv);
        s = s * exp2f((m - nm) * kLog2e) + exp2f((v.x - nm) * kLog2e) + exp2f((v.y - nm) * kLog2e) +
            exp2f((v.z - nm) * kLog2e) + exp2f((v.w - nm) * kLog2e);
        m = nm;
    }
    const float gm = block_reduce<true>(m, red);
    s = s * exp2f((m - gm) * kLog2e);
    const float gs = block_reduce<false>(s, red);
    const float inv = 1.f / gs;
    const float mb = gm * kLog2e;
    for (long long k = threadIdx.x; k < nvec; k += kThreads) {
        float4 v = xr[k];
        v.x = exp2f(fmaf(v.x, kLog2e, -mb)) * inv;
        v.y = exp2f(fmaf(v.y, kLog2e, -mb)) * inv;
        v.z = exp2f(fmaf(v.z, kLog2e, -mb)) * inv;
        v.w = exp2f(fmaf(v.w, kLog2e, -mb)) * inv;
        st_stream(yr + k, v);
    }
}

// any row length / 4-byte alignment: scalar accesses, online (max, sum), then normalise
__global__ void __launch_bounds__(kThreads) softmax_rows_scalar(const float* __restrict__ x,
                                                                float* __restrict__ y, long long cols) {
    __shared__ float red[kThreads / 32];
    const float* xr = x + (long long)blockIdx.x * cols;
    float* yr = y + (long long)blockIdx.x * cols;
    float m = -INFINITY, s = 0.f;
    for (long long k = threadIdx.x; k < cols; k += kThreads) {
        const float v = xr[k];
        const float nm = fmaxf(m, v);
        s = s * exp2f((m - nm) * kLog2e) + exp2f((v - nm) * kLog2e);
        m = nm;
    }
    const float gm = block_reduce<true>(m, red);
    s = m == -INFINITY ? 0.f : s * exp2f((m - gm) * kLog2e);
    const float inv = 1.f / block_reduce<false>(s, red);
    const float mb = gm * kLog2e;
    for (long long k = threadIdx.x; k < cols; k += kThreads) yr[k] = exp2f(fmaf(xr[k], kLog2e, -mb)) * inv;
}

}  // namespace

extern "C" lego_status lego_softmax_f32(const float* x, float* y, int64_t rows, int64_t cols,
                                        void* stream) {
    if (rows < 0 || cols <= 0) return lego_fail(LEGO_E_SHAPE, "bad softmax shape %lld x %lld",
                                                (long long)rows, (long long)cols);
    if (rows == 0) return LEGO_OK;
    if (!x || !y) return lego_fail(LEGO_E_ARG, "null buffer");
    if (((uintptr_t)x | (uintptr_t)y) & 3) return lego_fail(LEGO_E_ARG, "buffers must be 4-byte aligned");
    if (rows > 0x7fffffffLL) return lego_fail(LEGO_E_SHAPE, "too many rows");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (cols % 4 || (((uintptr_t)x | (uintptr_t)y) & 15)) {   // ragged rows: scalar path
        softmax_rows_scalar<<<(unsigned)rows, kThreads, 0, st>>>(x, y, cols);
        return lego_cuda_check(cudaGetLastError(), "softmax launch");
    }
    const long long per_pass = 4LL * kThreads;                  // floats per register "it"
    const long long its = (cols + per_pass - 1) / per_pass;
    dim3 grid((unsigned)rows);
    if (its <= 1) softmax_rows_reg<1><<<grid, kThreads, 0, st>>>(x, y, cols);
    else if (its <= 2) softmax_rows_reg<2><<<grid, kThreads, 0, st>>>(x, y, cols);
    else if (its <= 4) softmax_rows_reg<4><<<grid, kThreads, 0, st>>>(x, y, cols);
    else if (its <= 8) softmax_rows_reg<8><<<grid, kThreads, 0, st>>>(x, y, cols);
    else if (its <= 16) softmax_rows_reg<16><<<grid, kThreads, 0, st>>>(x, y, cols);
    else softmax_rows_stream<<<grid, kThreads, 0, st>>>(x, y, cols);
    return lego_cuda_check(cudaGetLastError(), "softmax launch");
}
