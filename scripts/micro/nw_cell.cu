// NW step micro-benchmark: one warp runs the compute warp's 4x4-cell step
// (lane j owns 4 columns, 4 rows per step, left column by SHFL.UP from lane
// j-1, offset-score recurrence), with the cell arithmetic written four ways:
//   A  IADD3(diag, sim, 2p) + VIMNMX3(., up, left)         (the kernel today)
//   B  IADD(diag, sim')      + VIMNMX3                      (sim' = sim + 2p pre-added)
//   C  FADD(diag, sim'_f)    + VIMNMX3 on the bits           (biased floats: x + 2^23 as fp32,
//                                                              integer-valued, bit order = value order)
//   D  VIADDMNMX(diag, sim', up) + VIMNMX(., left)          (DPX __viaddmax_s32)
//   E  sim' as packed fp16 pairs (2 LDS.128 per step instead of 4), FHADD(half, biased float) + VIMNMX3
// and optionally with the shared-memory traffic of the real step (4 LDS.128
// sim rows, 4 STS.128 S' rows).  Prints cycles per step (clock64, one warp).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o nw_cell nw_cell.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int V, int SMEM>   // SMEM bit 0: LDS of sim (prefetched two steps ahead), bit 1: STS of S'
__global__ void step_kernel(const int* in, int* out, long long* cyc, int steps) {
    __shared__ int4 ring[64 * 32];
    const int lane = threadIdx.x;
    for (int i = lane; i < 64 * 32; i += 32) ring[i] = make_int4(in[i & 255], in[(i + 1) & 255], in[(i + 2) & 255], in[(i + 3) & 255]);
    __syncwarp();
    int h[4], send[4], lin[4];
    for (int q = 0; q < 4; ++q) h[q] = send[q] = lin[q] = 0;
    int d = 0;
    const int p2 = 20;
    int4 s0 = make_int4(in[lane], in[lane + 1], in[lane + 2], in[lane + 3]);
    int4 s1 = make_int4(in[lane + 4], in[lane + 5], in[lane + 6], in[lane + 7]);
    int4 s2 = make_int4(in[lane + 8], in[lane + 9], in[lane + 10], in[lane + 11]);
    int4 s3 = make_int4(in[lane + 12], in[lane + 13], in[lane + 14], in[lane + 15]);
    if (V == 2 || V == 4) {   // biased floats
        for (int q = 0; q < 4; ++q) { h[q] = __float_as_int(8388608.0f); send[q] = lin[q] = h[q]; }
        d = h[0];
    }
    __shared__ unsigned tmem_base;
    unsigned tm = 0;
    if (V == 5) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;"
                     :: "r"((unsigned)__cvta_generic_to_shared(&tmem_base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncwarp();
        asm volatile("tcgen05.fence::after_thread_sync;");
        tm = tmem_base;
        unsigned w[16];
        for (int i = 0; i < 16; ++i) w[i] = (unsigned)in[(lane + i) & 255];
        for (int b = 0; b < 2; ++b)
            asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                         :: "r"(tm + 16 * b), "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]),
                            "r"(w[7]), "r"(w[8]), "r"(w[9]), "r"(w[10]), "r"(w[11]), "r"(w[12]), "r"(w[13]), "r"(w[14]),
                            "r"(w[15]));
        asm volatile("tcgen05.wait::st.sync.aligned;");
    }
    unsigned tv[16];
    if (V == 5) {
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                     : "=r"(tv[0]), "=r"(tv[1]), "=r"(tv[2]), "=r"(tv[3]), "=r"(tv[4]), "=r"(tv[5]), "=r"(tv[6]), "=r"(tv[7]),
                       "=r"(tv[8]), "=r"(tv[9]), "=r"(tv[10]), "=r"(tv[11]), "=r"(tv[12]), "=r"(tv[13]), "=r"(tv[14]), "=r"(tv[15])
                     : "r"(tm));
    }
    int4 nx1[4], nx2[4];
    for (int q = 0; q < 4; ++q) { nx1[q] = ring[q * 32 + lane]; nx2[q] = ring[(q + 4) * 32 + lane]; }
    long long t0 = clock64();
#pragma unroll 1
    for (int s8 = 0; s8 < steps; s8 += 8)
#pragma unroll
    for (int s = s8; s < s8 + 8; ++s) {
        int4 cur[4];
        if (V == 5) {
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            cur[0] = make_int4(tv[0], tv[1], tv[2], tv[3]);
            cur[1] = make_int4(tv[4], tv[5], tv[6], tv[7]);
            cur[2] = make_int4(tv[8], tv[9], tv[10], tv[11]);
            cur[3] = make_int4(tv[12], tv[13], tv[14], tv[15]);
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                         : "=r"(tv[0]), "=r"(tv[1]), "=r"(tv[2]), "=r"(tv[3]), "=r"(tv[4]), "=r"(tv[5]), "=r"(tv[6]), "=r"(tv[7]),
                           "=r"(tv[8]), "=r"(tv[9]), "=r"(tv[10]), "=r"(tv[11]), "=r"(tv[12]), "=r"(tv[13]), "=r"(tv[14]), "=r"(tv[15])
                         : "r"(tm + 16 * ((s + 1) & 1)));
        } else if (V == 4) {
            // two rows per 16-byte load: row q in .x/.y (q even) or .z/.w (q odd)
            const int row = (s * 4 + lane * 4) & 63;
            int4 a, b;
            if (SMEM & 1) {
                a = nx1[0]; b = nx1[1];
                nx1[0] = nx2[0]; nx1[1] = nx2[1];
                nx2[0] = ring[((row + 8) & 63) * 32 + lane];
                nx2[1] = ring[((row + 10) & 63) * 32 + lane];
            } else {
                a = s0; b = s1;
                s0.x ^= s; s1.y ^= s;
            }
            cur[0] = make_int4(a.x, a.y, 0, 0);
            cur[1] = make_int4(a.z, a.w, 0, 0);
            cur[2] = make_int4(b.x, b.y, 0, 0);
            cur[3] = make_int4(b.z, b.w, 0, 0);
        } else if (SMEM & 1) {
            const int row = (s * 4 + lane * 4) & 63;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                cur[q] = nx1[q];
                nx1[q] = nx2[q];
                nx2[q] = ring[((row + q + 8) & 63) * 32 + lane];
            }
        } else {
            cur[0] = s0; cur[1] = s1; cur[2] = s2; cur[3] = s3;
            s0.x ^= s; s1.y ^= s; s2.z ^= s; s3.w ^= s;   // keep the sim operands live and varying
        }
        int up0 = h[0], up1 = h[1], up2 = h[2], up3 = h[3];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int left = lane == 0 ? (s & 7) : lin[q];
            int x0, x1, x2, x3;
            if (V == 0) {
                x0 = max(max(cur[q].x + d + p2, up0), left);
                x1 = max(max(cur[q].y + up0 + p2, up1), x0);
                x2 = max(max(cur[q].z + up1 + p2, up2), x1);
                x3 = max(max(cur[q].w + up2 + p2, up3), x2);
            } else if (V == 1) {
                x0 = max(max(cur[q].x + d, up0), left);
                x1 = max(max(cur[q].y + up0, up1), x0);
                x2 = max(max(cur[q].z + up1, up2), x1);
                x3 = max(max(cur[q].w + up2, up3), x2);
            } else if (V == 2) {
                x0 = max(max(__float_as_int(__fadd_rn(__int_as_float(d), __int_as_float(cur[q].x))), up0), left);
                x1 = max(max(__float_as_int(__fadd_rn(__int_as_float(up0), __int_as_float(cur[q].y))), up1), x0);
                x2 = max(max(__float_as_int(__fadd_rn(__int_as_float(up1), __int_as_float(cur[q].z))), up2), x1);
                x3 = max(max(__float_as_int(__fadd_rn(__int_as_float(up2), __int_as_float(cur[q].w))), up3), x2);
            } else if (V == 4) {
                float f0, f1, f2, f3;
                asm("{\n\t.reg .f16 lo, hi;\n\tmov.b32 {lo, hi}, %2;\n\tadd.rn.f32.f16 %0, lo, %3;\n\tadd.rn.f32.f16 %1, hi, %4;\n\t}"
                    : "=f"(f0), "=f"(f1) : "r"(cur[q].x), "f"(__int_as_float(d)), "f"(__int_as_float(up0)));
                asm("{\n\t.reg .f16 lo, hi;\n\tmov.b32 {lo, hi}, %2;\n\tadd.rn.f32.f16 %0, lo, %3;\n\tadd.rn.f32.f16 %1, hi, %4;\n\t}"
                    : "=f"(f2), "=f"(f3) : "r"(cur[q].y), "f"(__int_as_float(up1)), "f"(__int_as_float(up2)));
                x0 = max(max(__float_as_int(f0), up0), left);
                x1 = max(max(__float_as_int(f1), up1), x0);
                x2 = max(max(__float_as_int(f2), up2), x1);
                x3 = max(max(__float_as_int(f3), up3), x2);
            } else if (V == 5) {
                x0 = max(max(cur[q].x + d + p2, up0), left);
                x1 = max(max(cur[q].y + up0 + p2, up1), x0);
                x2 = max(max(cur[q].z + up1 + p2, up2), x1);
                x3 = max(max(cur[q].w + up2 + p2, up3), x2);
            } else {
                x0 = max(__viaddmax_s32(d, cur[q].x, up0), left);
                x1 = max(__viaddmax_s32(up0, cur[q].y, up1), x0);
                x2 = max(__viaddmax_s32(up1, cur[q].z, up2), x1);
                x3 = max(__viaddmax_s32(up2, cur[q].w, up3), x2);
            }
            if (SMEM & 4) {   // S' row to tensor memory (lane j's TMEM lane), 4 columns per row
                asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};"
                             :: "r"(tm + 32 + 16 * (s & 1) + 4 * q), "r"(x0), "r"(x1), "r"(x2), "r"(x3));
            } else if (SMEM & 2) ring[((s * 4 + lane * 4 + q + 32) & 63) * 32 + lane] = make_int4(x0, x1, x2, x3);
            up0 = x0; up1 = x1; up2 = x2; up3 = x3;
            d = left;
            send[q] = x3;
            lin[q] = __shfl_up_sync(0xffffffffu, send[q], 1);
        }
        h[0] = up0; h[1] = up1; h[2] = up2; h[3] = up3;
    }
    long long t1 = clock64();
    if (lane == 0) cyc[0] = t1 - t0;
    if (V == 5) {
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        asm volatile("tcgen05.wait::st.sync.aligned;");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" :: "r"(tm));
    }
    __syncwarp();
    out[lane] = h[0] ^ h[1] ^ h[2] ^ h[3] ^ d ^ ring[(lane * 37) & 2047].x ^ ring[(steps + lane) & 2047].w;
}

template <int V, int SMEM>
double run(const int* in, int* out, long long* cyc, int steps) {
    step_kernel<V, SMEM><<<1, 32>>>(in, out, cyc, steps);
    cudaDeviceSynchronize();
    long long h;
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    return (double)h / steps;
}

int main() {
    int *in, *out;
    long long* cyc;
    cudaMalloc(&in, 4096);
    cudaMalloc(&out, 4096);
    cudaMalloc(&cyc, 64);
    int h_in[1024];
    for (int i = 0; i < 1024; ++i) h_in[i] = (i * 7) % 21 - 10;
    cudaMemcpy(in, h_in, 4096, cudaMemcpyHostToDevice);
    const int steps = 100000;
    const char* names[4] = {"registers only", "+ LDS (prefetched)", "+ STS", "+ LDS + STS"};
    for (int rep = 0; rep < 2; ++rep) {
        double r[4][5] = {{run<0, 0>(in, out, cyc, steps), run<1, 0>(in, out, cyc, steps), run<2, 0>(in, out, cyc, steps), run<3, 0>(in, out, cyc, steps), run<4, 0>(in, out, cyc, steps)},
                          {run<0, 1>(in, out, cyc, steps), run<1, 1>(in, out, cyc, steps), run<2, 1>(in, out, cyc, steps), run<3, 1>(in, out, cyc, steps), run<4, 1>(in, out, cyc, steps)},
                          {run<0, 2>(in, out, cyc, steps), run<1, 2>(in, out, cyc, steps), run<2, 2>(in, out, cyc, steps), run<3, 2>(in, out, cyc, steps), run<4, 2>(in, out, cyc, steps)},
                          {run<0, 3>(in, out, cyc, steps), run<1, 3>(in, out, cyc, steps), run<2, 3>(in, out, cyc, steps), run<3, 3>(in, out, cyc, steps), run<4, 3>(in, out, cyc, steps)}};
        for (int m = 0; m < 4; ++m)
            printf("cycles per 4x4 step, %-20s A %.1f  B %.1f  C %.1f  D %.1f  E %.1f\n", names[m], r[m][0], r[m][1], r[m][2], r[m][3], r[m][4]);
        printf("F (sim from TMEM, tcgen05.ld.32x32b.x16 a step ahead): registers only %.1f, + STS %.1f, + S' by tcgen05.st %.1f\n",
               run<5, 0>(in, out, cyc, steps), run<5, 2>(in, out, cyc, steps), run<5, 4>(in, out, cyc, steps));
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("err %s\n", cudaGetErrorString(e));
    return 0;
}
