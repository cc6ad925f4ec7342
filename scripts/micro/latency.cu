// Latency micro-benchmarks (one warp): dependent chains of SHFL, 3-input max,
// IADD3, LDS, and the NW step's shuffle->select->max pattern.  nvcc -arch=sm_100a
#include <cstdio>
#include <cuda_runtime.h>

__global__ void lat(int* out, long long* cyc, int iters, int seed) {
    __shared__ int sm[1024];
    const int lane = threadIdx.x;
    for (int i = lane; i < 1024; i += 32) sm[i] = (i * 7 + seed) & 1023;
    __syncwarp();
    int x = lane + seed, y = seed * 3, z = lane ^ seed;
    long long t0, t1;
    // 1. SHFL chain
    t0 = clock64();
    for (int i = 0; i < iters; ++i) x = __shfl_up_sync(0xffffffffu, x, 1) ^ i;
    t1 = clock64();
    if (lane == 0) cyc[0] = (t1 - t0);
    // 2. max3 chain
    t0 = clock64();
    for (int i = 0; i < iters; ++i) { y = max(max(y, z), x) ; z = max(max(z + 1, y), i); }
    t1 = clock64();
    if (lane == 0) cyc[1] = (t1 - t0);
    // 3. iadd3 chain
    t0 = clock64();
    for (int i = 0; i < iters; ++i) { y = y + z + i; z = z + y + x; }
    t1 = clock64();
    if (lane == 0) cyc[2] = (t1 - t0);
    // 4. LDS chain (pointer chase)
    int p = lane;
    t0 = clock64();
    for (int i = 0; i < iters; ++i) p = sm[p];
    t1 = clock64();
    if (lane == 0) cyc[3] = (t1 - t0);
    // 5. NW-like: shfl -> sel -> max3 -> shfl
    int v = lane, b = seed;
    t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        int l = __shfl_up_sync(0xffffffffu, v, 1);
        l = lane == 0 ? b : l;
        v = max(max(v + i, l), y);
    }
    t1 = clock64();
    if (lane == 0) cyc[4] = (t1 - t0);
    // 6. shfl via smem (STS + bar-free LDS of neighbour)
    volatile int* vs = sm;
    int u = lane;
    t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        vs[lane + 32 * (i & 1)] = u;
        __syncwarp();
        u = vs[((lane + 31) & 31) + 32 * (i & 1)] + i;
    }
    t1 = clock64();
    if (lane == 0) cyc[5] = (t1 - t0);
    out[lane] = x + y + z + p + v + u;
}

int main() {
    int* out; long long* cyc;
    cudaMalloc(&out, 1024); cudaMallocManaged(&cyc, 64 * 8);
    const int iters = 4096;
    for (int rep = 0; rep < 2; ++rep) {
        lat<<<1, 32>>>(out, cyc, iters, rep);
        cudaDeviceSynchronize();
    }
    const char* names[] = {"shfl chain", "2x max3 chain (per iter: 2 dep max3 + add)", "2x iadd3 chain",
                           "lds pointer chase", "shfl->sel->max3 loop", "smem exchange (sts+syncwarp+lds)"};
    for (int k = 0; k < 6; ++k) printf("%-45s %.1f cycles/iter\n", names[k], (double)cyc[k] / iters);
    return 0;
}
