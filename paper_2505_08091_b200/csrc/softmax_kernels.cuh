// softmax_kernels.cuh -- row softmax, fp32, one CTA per row (BASELINE.json
// config 3).  Kernel template shared by the static library (softmax.cu,
// runtime cols) and the programs generated from the LEGO thread/data layout
// (kernels.softmax_program: NVRTC, `namespace gen` in front of this file).
//
// Thread/data layout (the paper's softmax, index ops 4 -> 0):
//     GroupBy([rows], [cols/(4T)], [T], [4]).OrderBy(Row(rows, cols))
// element (row, it, tid, v) lives at apply(row, it, tid, v); the generated
// gen::vec_of(row, it, tid, k) is apply(row, it, tid, 0) / 4 (a float4
// index, simplified to row*cols/4 + it*T + tid), so every warp access is a
// coalesced float4, and a row is held in registers: HBM sees one read and
// one write per element.  When a row does not fit the register budget the
// static kernel streams it twice (online max/sum, then the normalised write).
//
// Includer-provided switches:
//   SM_GEN  1: gen::vec_of and gen::ITS (float4 vectors per thread) exist,
//              cols = gen::COLS; lego_softmax_offsets dumps the offsets
#pragma once

#ifndef SM_GEN
#define SM_GEN 0
#endif
#ifndef SM_GLOBAL
#define SM_GLOBAL extern "C" __global__
#endif

namespace smk {

constexpr int kThreads = 256;
constexpr float kLog2e = 1.4426950408889634f;

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
    float r = lane < (kThreads / 32) ? red[lane] : (IsMax ? -__int_as_float(0x7f800000) : 0.f);
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

// float4 index of (row, it, tid): the layout's apply / 4
__device__ __forceinline__ long long vec_index(long long row, int it, int tid, long long cols) {
#if SM_GEN
    (void)cols;
    long long k;
    gen::vec_of(row, (long long)it, (long long)tid, k);
    return k;
#else
    return row * (cols >> 2) + (long long)it * kThreads + tid;
#endif
}

// IT = float4 vectors per thread: the whole row lives in registers
template <int IT>
__device__ __forceinline__ void softmax_reg_body(const float* __restrict__ x, float* __restrict__ y,
                                                 long long cols) {
    __shared__ float red[kThreads / 32];
    const long long row = blockIdx.x;
    const float4* x4 = reinterpret_cast<const float4*>(x);
    float4* y4 = reinterpret_cast<float4*>(y);
    const int nvec = (int)(cols >> 2);
    const float ninf = -__int_as_float(0x7f800000);
    float4 v[IT];
    float m = ninf;
#pragma unroll
    for (int it = 0; it < IT; ++it) {
        const bool in = it * kThreads + (int)threadIdx.x < nvec;
        v[it] = in ? ld_stream(x4 + vec_index(row, it, threadIdx.x, cols)) : make_float4(ninf, ninf, ninf, ninf);
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
        if (it * kThreads + (int)threadIdx.x < nvec)
            st_stream(y4 + vec_index(row, it, threadIdx.x, cols),
                      make_float4(v[it].x * inv, v[it].y * inv, v[it].z * inv, v[it].w * inv));
    }
}

}  // namespace smk

#if SM_GEN
SM_GLOBAL void __launch_bounds__(smk::kThreads) lego_softmax_rows(const float* __restrict__ x,
                                                                  float* __restrict__ y) {
    smk::softmax_reg_body<gen::ITS>(x, y, gen::COLS);
}

// the float offsets the kernel reads and writes, for the layout check:
// out[(row*ITS + it)*T + tid] = 4 * vec_of(row, it, tid) (-1 past the row)
SM_GLOBAL void lego_softmax_offsets(long long* __restrict__ out) {
    const long long row = blockIdx.x;
    for (int it = 0; it < gen::ITS; ++it) {
        const bool in = it * smk::kThreads + (int)threadIdx.x < (int)(gen::COLS >> 2);
        out[(row * gen::ITS + it) * smk::kThreads + threadIdx.x] =
            in ? 4 * smk::vec_index(row, it, threadIdx.x, gen::COLS) : -1;
    }
}
#endif
