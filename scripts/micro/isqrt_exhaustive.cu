// Exhaustive check of lego_isqrt32 (csrc/lego_index.cuh) over [0, 2^31) plus
// negative arguments: r*r <= x < (r+1)^2 in 64-bit arithmetic, 0 for x <= 0.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2505_08091_b200/csrc \
//        scripts/micro/isqrt_exhaustive.cu -o /tmp/isqrt && /tmp/isqrt
#include <cstdio>
#include "lego_index.cuh"

__global__ void check(unsigned long long* bad, long long lo, long long hi) {
    unsigned long long local = 0;
    for (long long x = lo + blockIdx.x * (long long)blockDim.x + threadIdx.x; x < hi;
         x += (long long)gridDim.x * blockDim.x) {
        const long long r = lego_isqrt32((int)x);
        const bool ok = x <= 0 ? r == 0 : (r * r <= x && (r + 1) * (r + 1) > x);
        local += !ok;
    }
    if (local) atomicAdd(bad, local);
}

int main() {
    unsigned long long* bad;
    cudaMallocManaged(&bad, sizeof *bad);
    *bad = 0;
    check<<<148 * 16, 256>>>(bad, 0, 1LL << 31);
    check<<<148 * 16, 256>>>(bad, -(1LL << 31), -(1LL << 31) + (1LL << 24));
    check<<<148 * 16, 256>>>(bad, -(1LL << 24), 0);
    cudaDeviceSynchronize();
    printf("isqrt32 mismatches over [0, 2^31) and 2^25 negatives: %llu\n", *bad);
    return *bad != 0;
}
