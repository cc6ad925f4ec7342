// tma_transpose.cu -- micro-benchmark: TMA-staged 2-D transpose of a
// 16384 x 16384 bf16 matrix on B200 (and a TMA box copy for reference).
//
// Each warp is independent: lane 0 streams 64 x 64 source boxes into an
// S-slot ring (cp.async.bulk.tensor.2d, SWIZZLE_128B, mbarrier complete_tx),
// the warp transposes a box through registers (16-byte LDS of 8 x 8
// micro-tiles, __byte_perm transpose, 16-byte STS into a D-slot store ring
// in the destination's swizzled order), and lane 0 writes it back with a
// TMA store (cp.async.bulk.tensor.2d.global.shared, bulk async-groups).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_transpose tma_transpose.cu -lcuda
//   ./tma_transpose            (prints GB/s per variant and checks the result)
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#define CK(x)                                                                                     \
    do {                                                                                          \
        cudaError_t e_ = (x);                                                                     \
        if (e_ != cudaSuccess) {                                                                  \
            printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));                     \
            exit(1);                                                                              \
        }                                                                                         \
    } while (0)

constexpr int N = 16384;
constexpr int BOX = 64;                 // 64 x 64 bf16 = 8 KiB, rows of 128 B
constexpr int BOX_BYTES = BOX * BOX * 2;

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}"
        :: "r"(bar), "r"(parity) : "memory");
}
__device__ __forceinline__ void tma_load_2d(unsigned dst, const CUtensorMap* map, unsigned bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
        :: "r"(dst), "l"(map), "r"(bar), "r"(c0), "r"(c1) : "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, unsigned src, int c0, int c1) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];"
                 :: "l"(map), "r"(src), "r"(c0), "r"(c1) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int K>
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;" :: "n"(K) : "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

struct V16 { unsigned w[4]; };
__device__ __forceinline__ V16 lds16(unsigned a) {
    V16 v;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.w[0]), "=r"(v.w[1]), "=r"(v.w[2]), "=r"(v.w[3]) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts16(unsigned a, const V16& v) {
    asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" :: "r"(a), "r"(v.w[0]), "r"(v.w[1]), "r"(v.w[2]), "r"(v.w[3])
                 : "memory");
}

// transpose of an 8 x 8 bf16 block held as 8 rows of 16 bytes
__device__ __forceinline__ void tr8(const V16 (&in)[8], V16 (&out)[8]) {
#pragma unroll
    for (int c = 0; c < 8; ++c)
#pragma unroll
        for (int w = 0; w < 4; ++w)
            out[c].w[w] = __byte_perm(in[2 * w].w[c >> 1], in[2 * w + 1].w[c >> 1], (c & 1) ? 0x7632 : 0x5410);
}

// MODE 0: TMA copy (box in -> box out, same coordinates); MODE 1: transpose
template <int W, int S, int D, int MODE>
__global__ void __launch_bounds__(W * 32, 1) tma_kernel(const __grid_constant__ CUtensorMap src_map,
                                                        const __grid_constant__ CUtensorMap dst_map, int order) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<size_t>(smem_raw) + 1023) & ~size_t(1023));
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned char* wbase = smem + (size_t)warp * (S + D) * BOX_BYTES;
    const unsigned sbuf = smem_u32(wbase);
    const unsigned dbuf = sbuf + S * BOX_BYTES;
    unsigned long long* bars = reinterpret_cast<unsigned long long*>(smem + (size_t)W * (S + D) * BOX_BYTES) + warp * S;
    const unsigned bar0 = smem_u32(bars);
    constexpr int NT = N / BOX;                       // tiles per side
    const int total = NT * NT;
    const int gw = blockIdx.x * W + warp, nw = gridDim.x * W;
    const int count = gw < total ? (total - gw + nw - 1) / nw : 0;
    auto tile = [&](int k, int& tx, int& ty) {       // k-th tile of this warp
        const int t = gw + k * nw;
        if (order == 0) { tx = t % NT; ty = t / NT; }
        else if (order == 1) { ty = t % NT; tx = t / NT; }
        else {                                        // 8 x 8 blocks of tiles, x fastest inside
            const int blk = t / 64, in = t % 64;
            tx = (blk % (NT / 8)) * 8 + in % 8;
            ty = (blk / (NT / 8)) * 8 + in / 8;
        }
    };
    if (lane == 0) {
        for (int s = 0; s < S; ++s) mbar_init(bar0 + 8 * s, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int k = 0; k < S && k < count; ++k) {
            int tx, ty;
            tile(k, tx, ty);
            mbar_expect_tx(bar0 + 8 * k, BOX_BYTES);
            tma_load_2d(sbuf + k * BOX_BYTES, &src_map, bar0 + 8 * k, ty * BOX, tx * BOX);   // {col, row}
        }
    }
    __syncwarp();
    for (int k = 0; k < count; ++k) {
        const int s = k % S, ds = k % D;
        int tx, ty;
        tile(k, tx, ty);
        mbar_wait(bar0 + 8 * s, (k / S) & 1);
        const unsigned sb = sbuf + s * BOX_BYTES;
        if (MODE == 0) {
            // copy: store the landed box straight back out
            if (lane == 0) {
                tma_store_2d(&dst_map, sb, ty * BOX, tx * BOX);
                bulk_commit();
            }
        } else {
            const unsigned db = dbuf + ds * BOX_BYTES;
            if (lane == 0) bulk_wait_read<D - 1>();  // the store issued D tiles ago has read this slot
            __syncwarp();
            const int yc = lane & 7;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int xc = (((lane >> 3) << 1) + h + yc) & 7;
                V16 in[8], out[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) in[i] = lds16(sb + (8 * xc + i) * 128 + ((yc ^ i) << 4));
                tr8(in, out);
#pragma unroll
                for (int m = 0; m < 8; ++m) sts16(db + (8 * yc + m) * 128 + ((xc ^ m) << 4), out[m]);
            }
            fence_async_smem();
            __syncwarp();
            if (lane == 0) {
                tma_store_2d(&dst_map, db, tx * BOX, ty * BOX);                                // dst row = y
                bulk_commit();
            }
        }
        __syncwarp();
        if (lane == 0 && k + S < count) {
            int nx, ny;
            tile(k + S, nx, ny);
            if (MODE == 0) bulk_wait_read<0>();       // copy: the slot's own store must have read it
            fence_async_smem();
            mbar_expect_tx(bar0 + 8 * s, BOX_BYTES);
            tma_load_2d(sb, &src_map, bar0 + 8 * s, ny * BOX, nx * BOX);
        }
    }
    if (lane == 0) bulk_wait_all();
}

__global__ void ref_transpose(const unsigned short* __restrict__ a, unsigned short* __restrict__ b) {
    const long long i = blockIdx.y, j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    b[j * N + i] = a[i * N + j];
}
__global__ void count_diff(const unsigned short* a, const unsigned short* b, long long n, unsigned long long* bad) {
    unsigned long long c = 0;
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x)
        c += a[k] != b[k];
    if (c) atomicAdd(bad, c);
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static void make_map(EncodeFn enc, CUtensorMap* m, void* base, CUtensorMapL2promotion promo) {
    cuuint64_t dims[2] = {N, N};
    cuuint64_t strides[1] = {(cuuint64_t)N * 2};
    cuuint32_t box[2] = {BOX, BOX};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); exit(1); }
}

template <int W, int S, int D, int MODE>
static void run(EncodeFn enc, void* a, void* b, void* ref, int blocks_per_sm, int order, int promo) {
    CUtensorMap ms, md;
    const CUtensorMapL2promotion p = promo == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE
                                   : promo == 1 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
    make_map(enc, &ms, a, p);
    make_map(enc, &md, b, p);
    const int smem = W * (S + D) * BOX_BYTES + W * S * 8 + 1024;
    CK(cudaFuncSetAttribute(tma_kernel<W, S, D, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int grid = sms * blocks_per_sm;
    CK(cudaMemset(b, 0, (size_t)N * N * 2));
    tma_kernel<W, S, D, MODE><<<grid, W * 32, smem>>>(ms, md, order);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    unsigned long long* bad;
    CK(cudaMalloc(&bad, 8));
    CK(cudaMemset(bad, 0, 8));
    count_diff<<<1024, 256>>>((const unsigned short*)b, (const unsigned short*)(MODE ? ref : a), (long long)N * N, bad);
    unsigned long long hbad = 0;
    CK(cudaMemcpy(&hbad, bad, 8, cudaMemcpyDeviceToHost));
    cudaFree(bad);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int it = 50;
    for (int k = 0; k < 5; ++k) tma_kernel<W, S, D, MODE><<<grid, W * 32, smem>>>(ms, md, order);
    cudaEventRecord(e0);
    for (int k = 0; k < it; ++k) tma_kernel<W, S, D, MODE><<<grid, W * 32, smem>>>(ms, md, order);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms_ = 0;
    cudaEventElapsedTime(&ms_, e0, e1);
    const double us = ms_ * 1e3 / it;
    printf("%s W=%d S=%d D=%d ctas/SM=%d order=%d promo=%d smem=%d: %8.1f us %7.1f GB/s  mismatches=%llu\n",
           MODE ? "transpose" : "copy     ", W, S, D, blocks_per_sm, order, promo, smem, us,
           2.0 * N * N * 2 / us / 1e3, hbad);
}

int main() {
    void* a;
    void* b;
    void* ref;
    CK(cudaMalloc(&a, (size_t)N * N * 2));
    CK(cudaMalloc(&b, (size_t)N * N * 2));
    CK(cudaMalloc(&ref, (size_t)N * N * 2));
    std::vector<unsigned short> h((size_t)N * N);
    for (size_t k = 0; k < h.size(); ++k) h[k] = (unsigned short)(k * 2654435761u >> 7);
    CK(cudaMemcpy(a, h.data(), h.size() * 2, cudaMemcpyHostToDevice));
    ref_transpose<<<dim3(N / 256, N), 256>>>((const unsigned short*)a, (unsigned short*)ref);
    CK(cudaDeviceSynchronize());
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    EncodeFn enc = (EncodeFn)fn;
    {   // device-to-device copy reference
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        for (int k = 0; k < 3; ++k) cudaMemcpy(b, a, (size_t)N * N * 2, cudaMemcpyDeviceToDevice);
        cudaEventRecord(e0);
        for (int k = 0; k < 20; ++k) cudaMemcpyAsync(b, a, (size_t)N * N * 2, cudaMemcpyDeviceToDevice);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms_ = 0;
        cudaEventElapsedTime(&ms_, e0, e1);
        printf("cudaMemcpy D2D: %8.1f us %7.1f GB/s\n", ms_ * 1e3 / 20, 2.0 * N * N * 2 / (ms_ * 1e3 / 20) / 1e3);
    }
    run<4, 4, 2, 0>(enc, a, b, ref, 1, 0, 0);
    run<4, 4, 2, 0>(enc, a, b, ref, 1, 2, 0);
    run<4, 4, 2, 1>(enc, a, b, ref, 1, 0, 0);
    run<4, 4, 2, 1>(enc, a, b, ref, 1, 1, 0);
    run<4, 4, 2, 1>(enc, a, b, ref, 1, 2, 0);
    run<4, 4, 2, 1>(enc, a, b, ref, 1, 2, 1);
    run<8, 2, 1, 1>(enc, a, b, ref, 1, 2, 0);
    run<2, 4, 2, 1>(enc, a, b, ref, 2, 2, 0);
    run<2, 8, 2, 1>(enc, a, b, ref, 1, 2, 0);
    run<6, 3, 1, 1>(enc, a, b, ref, 1, 2, 0);
    return 0;
}
