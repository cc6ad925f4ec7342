// Single-warp shared-memory instruction rates on the B200: cycles per
// STS.128 / STS.64 / STS.32 / LDS.128 (independent, conflict-free, 16 in flight)
// and STS.128 with the NW ring's skewed rows (lane j writes row 4j).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o smem_rate smem_rate.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(int* out, long long* cyc, int iters, const int4* __restrict__ g = nullptr, int same_smsp = 0) {
    if (same_smsp && ((threadIdx.x >> 5) & 3)) return;   // only warps 0, 4, 8, ... (SMSP 0) work
    __shared__ int4 buf[64 * 32];
    const int lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 64 * 32; i += blockDim.x) buf[i] = make_int4(i, i ^ 1, i ^ 2, i ^ 3);
    __syncthreads();
    int4 v = make_int4(lane, lane + 1, lane + 2, lane + 3);
    int acc = 0;
    long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            const int row = (i * 16 + u) & 63;
            if (MODE == 0) buf[row * 32 + lane] = v;                                    // STS.128, same row
            if (MODE == 1) buf[((row + 4 * lane) & 63) * 32 + lane] = v;                // STS.128, skewed rows
            if (MODE == 2) reinterpret_cast<int2*>(buf)[row * 64 + lane] = make_int2(v.x, v.y);   // STS.64
            if (MODE == 3) reinterpret_cast<int*>(buf)[row * 128 + lane] = v.x;          // STS.32
            if (MODE == 4) { int4 w = buf[((row + 4 * lane + acc) & 63) * 32 + lane]; acc += w.x ^ w.w; }   // LDS.128 skewed (dependent)
            if (MODE == 5) { int4 w = buf[((row + 4 * lane) & 63) * 32 + lane]; acc += w.x ^ w.w; }   // LDS.128 skewed
            if (MODE == 6) { int2 w = reinterpret_cast<int2*>(buf)[((row + 4 * lane) & 63) * 64 + 2 * lane]; acc += w.x ^ w.y; }   // LDS.64
            if (MODE == 7) { acc += __shfl_up_sync(0xffffffffu, v.x + u, 1); }   // SHFL (independent)
            if (MODE == 11) {   // LDS.128 by lane 0 only (predicated)
                int4 w = make_int4(0, 0, 0, 0);
                asm volatile("{\n\t.reg .pred q;\n\tsetp.eq.s32 q, %4, 0;\n\t@q ld.shared.v4.b32 {%0,%1,%2,%3}, [%5];\n\t}"
                             : "+r"(w.x), "+r"(w.y), "+r"(w.z), "+r"(w.w) : "r"(lane), "r"((unsigned)__cvta_generic_to_shared(&buf[row * 32])));
                acc += w.x ^ w.w;
            }
            if (MODE == 12) {   // STS.128 by lane 0 only (predicated)
                asm volatile("{\n\t.reg .pred q;\n\tsetp.eq.s32 q, %0, 0;\n\t@q st.shared.v4.b32 [%1], {%2,%3,%4,%5};\n\t}"
                             :: "r"(lane), "r"((unsigned)__cvta_generic_to_shared(&buf[row * 32])), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w));
            }
            if (MODE == 13) { int4 w = g[((row + 4 * lane) & 63) * 32 + lane]; acc += w.x ^ w.w; }   // LDG.128 (L1 hits)
            if (MODE == 14) { int4 w = __ldg(&g[((row + 4 * lane) & 63) * 32 + lane]); acc += w.x ^ w.w; }   // LDG.128.CONSTANT
            if (MODE == 15 && (u & 3) == 0) {   // step mix with sim from L1: 4 LDG.128 + 4 STS.128 + 4 SHFL
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int r2 = (row + 4 * lane + q) & 63;
                    int4 w = g[((r2 + 8) & 63) * 32 + lane];
                    acc += w.x ^ w.w;
                    buf[r2 * 32 + lane] = v;
                    acc += __shfl_up_sync(0xffffffffu, v.x + q, 1);
                }
            }
            // step-like mixes, per 4 iterations of u (one NW step): 4 LDS.128 + 4 stores + 4 SHFL
            if (MODE >= 8 && (u & 3) == 0) {
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int r2 = (row + 4 * lane + q) & 63;
                    int4 w = buf[((r2 + 8) & 63) * 32 + lane];
                    acc += w.x ^ w.w;
                    if (MODE == 8) buf[r2 * 32 + lane] = v;
                    if (MODE == 9) {
                        reinterpret_cast<int2*>(buf)[r2 * 64 + 2 * lane] = make_int2(v.x, v.y);
                        reinterpret_cast<int2*>(buf)[r2 * 64 + 2 * lane + 1] = make_int2(v.z, v.w);
                    }
                    if (MODE == 10 && q == 3) buf[r2 * 32 + lane] = v;
                    acc += __shfl_up_sync(0xffffffffu, v.x + q, 1);
                }
            }
            v.x += u;
        }
    }
    long long t1 = clock64();
    __syncwarp();
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
    out[threadIdx.x] = acc + buf[lane].x + v.x;
}

static int4* g_buf = nullptr;
template <int MODE>
double run(int* out, long long* cyc, int warps = 1, int same = 0) {
    const int iters = 20000;
    k<MODE><<<1, 32 * warps>>>(out, cyc, iters, g_buf, same);
    cudaDeviceSynchronize();
    long long h;
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    return (double)h / (iters * 16);
}

int main() {
    int* out;
    long long* cyc;
    cudaMalloc(&out, 4096);
    cudaMalloc(&cyc, 64);
    cudaMalloc(&g_buf, 64 * 32 * 16);
    cudaMemset(g_buf, 1, 64 * 32 * 16);
    for (int w : {1, 2, 4})
        printf("cycles/instr per warp (%d warps): STS.128 %.2f  STS.128 skewed %.2f  STS.64 %.2f  STS.32 %.2f  "
               "LDS.128 dep %.2f  LDS.128 %.2f  LDS.64 %.2f  SHFL %.2f\n", w,
               run<0>(out, cyc, w), run<1>(out, cyc, w), run<2>(out, cyc, w), run<3>(out, cyc, w), run<4>(out, cyc, w),
               run<5>(out, cyc, w), run<6>(out, cyc, w), run<7>(out, cyc, w));
    for (int rep = 0; rep < 2; ++rep)
        printf("LDG.128 L1-hit %.2f  LDG.128.nc %.2f cycles/instr; step mix with sim from L1 (4 LDG + 4 STS.128 + 4 SHFL) %.1f\n",
               run<13>(out, cyc), run<14>(out, cyc), 4 * run<15>(out, cyc));
    for (int w : {4, 8, 12})
        printf("same SMSP, %d working warps: STS.128 %.2f  LDS.128 %.2f  SHFL %.2f cycles/instr per warp\n", w / 4 + 1,
               run<0>(out, cyc, w + 1, 1), run<5>(out, cyc, w + 1, 1), run<7>(out, cyc, w + 1, 1));
    printf("1-lane LDS.128 %.2f  1-lane STS.128 %.2f cycles/instr\n", run<11>(out, cyc), run<12>(out, cyc));
    for (int rep = 0; rep < 2; ++rep)
        printf("cycles per NW-like step (1 warp): 4 LDS.128 + 4 STS.128 + 4 SHFL %.1f | + 8 STS.64 instead %.1f | "
               "+ 1 STS.128 only %.1f\n", 4 * run<8>(out, cyc), 4 * run<9>(out, cyc), 4 * run<10>(out, cyc));
    return 0;
}
