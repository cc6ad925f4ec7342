// SM-to-SM hand-off latency (one-way = round trip / 2), the NW strip hand-off's
// floor: (1) global-memory flag ping-pong between two CTAs (relaxed gpu-scope
// store / polling load, the path lego_nw_tiles uses), per SM pair; (2) DSMEM
// ping-pong inside a 2-CTA cluster: remote st.shared::cluster + local polling;
// (3) st.async into the peer's shared memory completing a transaction on its
// mbarrier, the peer waiting on the mbarrier.  nvcc -arch=sm_100a -o handoff handoff.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>

namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ int ld_relaxed(const int* p) {
    int v;
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed(int* p, int v) {
    asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}

// (1) CTA 0 <-> CTA `peer` through two global flags
__global__ void pingpong_global(int* flags, int peer, int iters, unsigned long long* out, int* smids) {
    extern __shared__ int pad[];
    (void)pad;
    int sm;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
    if (threadIdx.x == 0) smids[blockIdx.x] = sm;
    if (threadIdx.x != 0 || (blockIdx.x != 0 && blockIdx.x != peer)) return;
    int* ping = flags;
    int* pong = flags + 64;
    if (blockIdx.x == 0) {
        // wait for the peer to be up
        while (ld_relaxed(pong) != -1) {}
        const unsigned long long t0 = gtime();
        for (int i = 1; i <= iters; ++i) {
            st_relaxed(ping, i);
            while (ld_relaxed(pong) != i) {}
        }
        out[0] = gtime() - t0;
    } else {
        st_relaxed(pong, -1);
        for (int i = 1; i <= iters; ++i) {
            while (ld_relaxed(ping) != i) {}
            st_relaxed(pong, i);
        }
    }
}

// (2) cluster of 2: remote store, local volatile poll
__global__ void __cluster_dims__(2, 1, 1) pingpong_dsmem(int iters, unsigned long long* out) {
    __shared__ int box[32];
    cg::cluster_group cl = cg::this_cluster();
    const unsigned r = cl.block_rank();
    if (threadIdx.x == 0) box[0] = 0;
    cl.sync();
    if (threadIdx.x == 0) {
        int* peer = cl.map_shared_rank(box, r ^ 1);
        volatile int* mine = box;
        const unsigned long long t0 = gtime();
        for (int i = 1; i <= iters; ++i) {
            if (r == 0) {
                asm volatile("st.relaxed.cluster.shared::cluster.b32 [%0], %1;" ::
                             "r"((unsigned)__cvta_generic_to_shared(peer) ), "r"(i) : "memory");
                while (mine[0] != i) {}
            } else {
                while (mine[0] != i) {}
                asm volatile("st.relaxed.cluster.shared::cluster.b32 [%0], %1;" ::
                             "r"((unsigned)__cvta_generic_to_shared(peer)), "r"(i) : "memory");
            }
        }
        if (r == 0) out[1] = gtime() - t0;
    }
    cl.sync();
}

// (3) cluster of 2: st.async into the peer's box, completing 4 bytes on its mbarrier
__global__ void __cluster_dims__(2, 1, 1) pingpong_stasync(int iters, unsigned long long* out) {
    __shared__ alignas(8) unsigned long long mbar;
    __shared__ int box[4];
    cg::cluster_group cl = cg::this_cluster();
    const unsigned r = cl.block_rank();
    const unsigned mb = (unsigned)__cvta_generic_to_shared(&mbar);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(mb) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    cl.sync();
    if (threadIdx.x == 0) {
        unsigned peer_box, peer_mb;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(peer_box)
                     : "r"((unsigned)__cvta_generic_to_shared(box)), "r"(r ^ 1));
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(peer_mb) : "r"(mb), "r"(r ^ 1));
        unsigned phase = 0;
        auto arm = [&]() {
            asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], 4;\n\t}"
                         :: "r"(mb) : "memory");
        };
        auto wait = [&]() {
            asm volatile("{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
                         "@!p bra W;\n\t}" :: "r"(mb), "r"(phase) : "memory");
            phase ^= 1;
        };
        auto send = [&](int v) {
            asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];"
                         :: "r"(peer_box), "r"(v), "r"(peer_mb) : "memory");
        };
        arm();
        cl.sync();   // both armed (thread 0 only reaches here; other threads are in the other sync)
        const unsigned long long t0 = gtime();
        for (int i = 1; i <= iters; ++i) {
            if (r == 0) {
                send(i);
                wait();
                arm();
            } else {
                wait();
                arm();
                send(i);
            }
        }
        if (r == 0) out[2] = gtime() - t0;
    } else {
        cl.sync();
    }
    cl.sync();
}

int main() {
    int* flags;
    unsigned long long* out;
    int* smids;
    cudaMalloc(&flags, 4096);
    cudaMalloc(&out, 64);
    cudaMalloc(&smids, 148 * 4);
    const int iters = 2000;
    const int smem = 200 * 1024;
    cudaFuncSetAttribute(pingpong_global, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int h_smids[148];
    printf("global flag ping-pong, one-way ns, CTA 0 vs peer (smids):\n");
    for (int peer = 1; peer < 148; peer += 7) {
        cudaMemset(flags, 0, 4096);
        pingpong_global<<<148, 32, smem>>>(flags, peer, iters, out, smids);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
        unsigned long long h;
        cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
        cudaMemcpy(h_smids, smids, sizeof h_smids, cudaMemcpyDeviceToHost);
        printf("  peer %3d  sm %3d <-> sm %3d : %7.1f ns\n", peer, h_smids[0], h_smids[peer], h / 2.0 / iters);
    }
    for (int rep = 0; rep < 3; ++rep) {
        pingpong_dsmem<<<2, 32>>>(iters, out);
        pingpong_stasync<<<2, 32>>>(iters, out);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
        unsigned long long h[3];
        cudaMemcpy(h, out, 24, cudaMemcpyDeviceToHost);
        printf("cluster DSMEM store + local poll: %7.1f ns one-way;  st.async + mbarrier: %7.1f ns one-way\n",
               h[1] / 2.0 / iters, h[2] / 2.0 / iters);
    }
    return 0;
}
