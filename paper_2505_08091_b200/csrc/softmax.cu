// softmax.cu -- row softmax, fp32, one CTA per row (BASELINE.json config 3):
// the library's built-in kernels.  The register-resident kernel is the
// template of softmax_kernels.cuh with the layout's offset written for a
// runtime row length; kernels.softmax runs the LEGO-generated program of
// the same template (offsets from GroupBy([rows],[cols/4T],[T],[4])
// .OrderBy(Row(rows, cols)), tests/test_softmax_layout.py) whenever the row
// length is a whole number of 4T-float passes.  Long rows stream twice
// (online max/sum, then the normalised write); ragged rows take a scalar
// kernel.
#include <cuda_runtime.h>

#include "lego_common.h"

#define SM_GLOBAL static __global__
#include "softmax_kernels.cuh"

namespace {

using smk::block_reduce;
using smk::kLog2e;
using smk::kThreads;
using smk::st_stream;

template <int IT>
__global__ void __launch_bounds__(kThreads) softmax_rows_reg(const float* __restrict__ x,
                                                             float* __restrict__ y, long long cols) {
    smk::softmax_reg_body<IT>(x, y, cols);
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
