// remap_kernels.cuh -- hand-written sm_100a kernel templates for LEGO layouts.
//
// A program's source is:  lego_index.cuh + a generated `namespace gen { ... }`
// (constants and device functions from paper_2505_08091_b200/codegen.py) +
// this file with LEGO_KIND / LEGO_ELEM defined.  The generated functions are
// the layout's index arithmetic (reference GroupBy.apply / inv,
// pkg/src/lego/layout.py:313-328, lowered and simplified); the templates
// own the memory access pattern.
//
//   LEGO_KIND 0  index maps:  lego_apply_map_*, lego_inv_map_*, lego_hist
//   LEGO_KIND 1  gather:      dst[f] = src[g(f)]; 16-byte vector stores, and
//                             16-byte vector loads when g is provably
//                             contiguous over each vector (LEGO_CONTIG)
//   LEGO_KIND 2  transpose:   g is a mixed-radix digit permutation whose
//                             dst-innermost and src-innermost digits differ:
//                             each lane moves a VxV micro-tile (V = 16/E) with
//                             16-byte loads along src rows and 16-byte stores
//                             along dst rows, transposed in registers
//   LEGO_KIND 3  band:        anti-diagonal band tiles staged through smem
//   LEGO_KIND 4  scatter:     dst[apply(x)] = src[x] into an injective layout
//   LEGO_KIND 5  staged:      each destination block reads one source box,
//                             staged through smem (staging.py's proof)
#pragma once

#define LEGO_GLOBAL extern "C" __global__

struct lego_v16 { unsigned int w[4]; };

// memory-access qualifiers (LEGO_LDV / LEGO_STV select cache hints; 0 = default)
#ifndef LEGO_LDV
#define LEGO_LDV 0
#endif
#ifndef LEGO_STV
#define LEGO_STV 0
#endif
#if LEGO_LDV == 1
#define LEGO_LDQ "ld.global.nc.L1::no_allocate.L2::256B.v4.u32"
#elif LEGO_LDV == 2
#define LEGO_LDQ "ld.global.nc.L1::no_allocate.L2::128B.v4.u32"
#elif LEGO_LDV == 3
#define LEGO_LDQ "ld.global.nc.L1::evict_first.L2::256B.v4.u32"
#else
#define LEGO_LDQ "ld.global.nc.L1::no_allocate.v4.u32"
#endif
#if LEGO_STV == 1
#define LEGO_STQ "st.global.cs.v4.u32"
#elif LEGO_STV == 2
#define LEGO_STQ "st.global.v4.u32"
#else
#define LEGO_STQ "st.global.L1::no_allocate.v4.u32"
#endif
static __device__ __forceinline__ lego_v16 lego_ld16(const unsigned char* p) {
    lego_v16 v;
    asm volatile(LEGO_LDQ " {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.w[0]), "=r"(v.w[1]), "=r"(v.w[2]), "=r"(v.w[3]) : "l"(p));
    return v;
}
static __device__ __forceinline__ void lego_st16(unsigned char* p, const lego_v16& v) {
    asm volatile(LEGO_STQ " [%0], {%1,%2,%3,%4};"
                 :: "l"(p), "r"(v.w[0]), "r"(v.w[1]), "r"(v.w[2]), "r"(v.w[3]) : "memory");
}

// element loads of the band kernel: no L2 sector promotion (measured: the
// 256-byte hint over-fetches along the diagonal runs, 6058 -> 5099 GB/s) and
// no L1::no_allocate (6058 -> 5289 GB/s)
// (plain __ldg: the band kernel's row and diagonal runs reuse L1 lines)
template <typename T>
static __device__ __forceinline__ T lego_lde(const T* p) { return __ldg(p); }

template <int E> struct lego_elem;
template <> struct lego_elem<1> { typedef unsigned char t; };
template <> struct lego_elem<2> { typedef unsigned short t; };
template <> struct lego_elem<4> { typedef unsigned int t; };
template <> struct lego_elem<8> { typedef unsigned long long t; };

#if LEGO_ROUTED
// routed destinations (fused remap + all-to-all over peer memory, shard.py):
// the kernel's dst argument is a device array of per-rank base pointers (the
// peers' symmetric buffers, NVLink-mapped); destination element v of the
// remap goes to buffer gen::route(v).peer at element offset .off.  The
// planner proved that every aligned 16-byte destination vector stays in one
// peer, contiguous and 16-byte aligned (kernels._routed_plan).
static __device__ __forceinline__ unsigned char* lego_route(unsigned char* table, long long v, int elem) {
    long long peer, off;
    gen::route(v, peer, off);
    unsigned char* base = reinterpret_cast<unsigned char* const*>(table)[peer];
    return base + off * elem;
}
#endif

// ---------------------------------------------------------------------------
#if LEGO_KIND == 0
// index maps: one thread per output element, int32 or int64 outputs.
template <typename T>
static __device__ __forceinline__ T lego_map_one(long long x, int which) {
    long long r;
    if (which == 0) gen::apply_fn(x, r);
    else            gen::inv_fn(x, r);
    return (T)r;
}
// G consecutive indices per thread (G/4 16-byte int32 stores, or twice as
// many for int64) when the output is 16-byte aligned; scalar tail.  The
// memory-bound apply maps use G = 4 (fully coalesced stores); the
// ALU-bound inverse maps G = 8 (more independent work per thread: +4 % on
// the anti-diagonal inverse, where the half-coalesced stores cost nothing)
template <typename T, int G>
static __device__ __forceinline__ void lego_map_body(T* out, long long first, long long count,
                                                     int which) {
    const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long stride = (long long)gridDim.x * blockDim.x;
    long long done = 0;
    if ((reinterpret_cast<unsigned long long>(out) & 15) == 0) {
        const long long nq = count / G;
        for (long long q = tid; q < nq; q += stride) {
            const long long x = first + G * q;
            T v[G];
#pragma unroll
            for (int u = 0; u < G; ++u) v[u] = lego_map_one<T>(x + u, which);
#pragma unroll
            for (int g = 0; g < G / 4; ++g) {
                T* o = out + G * q + 4 * g;
                if (sizeof(T) == 4) {
                    *reinterpret_cast<int4*>(o) = make_int4((int)v[4 * g], (int)v[4 * g + 1], (int)v[4 * g + 2],
                                                            (int)v[4 * g + 3]);
                } else {
                    *reinterpret_cast<longlong2*>(o) = make_longlong2((long long)v[4 * g], (long long)v[4 * g + 1]);
                    *reinterpret_cast<longlong2*>(o + 2) = make_longlong2((long long)v[4 * g + 2],
                                                                          (long long)v[4 * g + 3]);
                }
            }
        }
        done = nq * G;
    }
    for (long long k = done + tid; k < count; k += stride) out[k] = lego_map_one<T>(first + k, which);
}
LEGO_GLOBAL void __launch_bounds__(256) lego_apply_map_i32(int* out, long long first, long long count) {
    lego_map_body<int, 4>(out, first, count, 0);
}
LEGO_GLOBAL void __launch_bounds__(256) lego_apply_map_i64(long long* out, long long first, long long count) {
    lego_map_body<long long, 4>(out, first, count, 0);
}
#if LEGO_INV_RUNS
// Inverse of an n x n layout whose positions run contiguously along
// anti-diagonals (kernels.index_map_source proved
// apply(i+1, j-1) == apply(i, j) + 1 symbolically, lower.diagonal_runs_contiguous):
// position f+1 holds (i+1, j-1) while that cell exists, so a thread
// evaluates the generated inverse (isqrt and selects) once for its first
// position and steps along the run for the rest -- logical row-major index
// + (n - 1) per position -- re-evaluating only where a diagonal ends.  Four
// positions per thread keep each store instruction fully coalesced (eight,
// as two 16-byte stores per lane, write half sectors and lose ~40 %).
template <typename T, int G>
static __device__ __forceinline__ void lego_inv_runs_body(T* out, long long first, long long count) {
    constexpr long long NN = gen::RUN_N;
    const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long stride = (long long)gridDim.x * blockDim.x;
    long long done = 0;
    if ((reinterpret_cast<unsigned long long>(out) & 15) == 0) {
        const long long nq = count / G;
        for (long long q = tid; q < nq; q += stride) {
            const long long x = first + G * q;
            long long r;
            gen::inv_fn(x, r);
            const long long i = r / NN, j = r - i * NN;
            // cells after (i, j) on its diagonal: the run continues that far
            const long long run = j < NN - 1 - i ? j : NN - 1 - i;
            T* o = out + G * q;
            if (run >= G - 1) {
#pragma unroll
                for (int g = 0; g < G / 4; ++g) {
                    const long long b = r + (long long)(4 * g) * (NN - 1);
                    if (sizeof(T) == 4) {
                        *reinterpret_cast<int4*>(o + 4 * g) =
                            make_int4((int)b, (int)(b + (NN - 1)), (int)(b + 2 * (NN - 1)), (int)(b + 3 * (NN - 1)));
                    } else {
                        *reinterpret_cast<longlong2*>(o + 4 * g) = make_longlong2(b, b + (NN - 1));
                        *reinterpret_cast<longlong2*>(o + 4 * g + 2) =
                            make_longlong2(b + 2 * (NN - 1), b + 3 * (NN - 1));
                    }
                }
            } else {                                   // a diagonal ends inside the group (rare)
#pragma unroll 1
                for (int u = 0; u < G; ++u) o[u] = lego_map_one<T>(x + u, 1);
            }
        }
        done = nq * G;
    }
    for (long long k = done + tid; k < count; k += stride) out[k] = lego_map_one<T>(first + k, 1);
}
LEGO_GLOBAL void __launch_bounds__(256) lego_inv_map_i32(int* out, long long first, long long count) {
    lego_inv_runs_body<int, 4>(out, first, count);
}
LEGO_GLOBAL void __launch_bounds__(256) lego_inv_map_i64(long long* out, long long first, long long count) {
    lego_inv_runs_body<long long, 4>(out, first, count);
}
#else
LEGO_GLOBAL void __launch_bounds__(256) lego_inv_map_i32(int* out, long long first, long long count) {
    lego_map_body<int, 8>(out, first, count, 1);
}
LEGO_GLOBAL void __launch_bounds__(256) lego_inv_map_i64(long long* out, long long first, long long count) {
    lego_map_body<long long, 8>(out, first, count, 1);
}
#endif
// histogram of apply over the whole logical space (bijectivity proof)
LEGO_GLOBAL void __launch_bounds__(256) lego_hist(unsigned int* hist, long long count, long long n_out,
                                                  unsigned long long* bad) {
    long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (; k < count; k += stride) {
        long long r;
        gen::apply_fn(k, r);
        if (r >= 0 && r < n_out) atomicAdd(hist + r, 1u);
        else if (r != -1) atomicAdd(bad, 1ull);
    }
}
// violations: positions not hit exactly once (bijective), or hit more than
// once (at_most_once: injective-mode layouts leave positions unhit)
LEGO_GLOBAL void __launch_bounds__(256) lego_hist_check(const unsigned int* hist, long long n,
                                                        unsigned long long* bad, int at_most_once) {
    long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long stride = (long long)gridDim.x * blockDim.x;
    unsigned long long local = 0;
    for (; k < n; k += stride) local += at_most_once ? (hist[k] > 1u) : (hist[k] != 1u);
    for (int o = 16; o; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
    if ((threadIdx.x & 31) == 0 && local) atomicAdd(bad, local);
}
#endif

// ---------------------------------------------------------------------------
#if LEGO_KIND == 1
// gather: each thread owns VEC consecutive destination elements (16 bytes),
// UNROLL vectors per thread with all loads issued before the stores.
#define LEGO_VEC (16 / LEGO_ELEM)
#ifndef LEGO_UNROLL
#define LEGO_UNROLL 4
#endif
typedef lego_elem<LEGO_ELEM>::t lego_e;

static __device__ __forceinline__ lego_v16 lego_gather_vec(const unsigned char* src, long long f) {
    lego_v16 v;
#if LEGO_CONTIG
    long long s;
    gen::src_of(f, s);
    v = lego_ld16(src + s * LEGO_ELEM);
#else
    union { lego_e e[LEGO_VEC]; lego_v16 v; } u;
#pragma unroll
    for (int k = 0; k < LEGO_VEC; ++k) {
        long long s;
        gen::src_of(f + k, s);
#if LEGO_MASKED
        u.e[k] = s >= 0 ? __ldg(reinterpret_cast<const lego_e*>(src) + s) : (lego_e)0;
#else
        u.e[k] = __ldg(reinterpret_cast<const lego_e*>(src) + s);
#endif
    }
    v = u.v;
#endif
    return v;
}

#if LEGO_SCALAR
// ragged sizes / unaligned batch strides: one element per thread, grid-stride
LEGO_GLOBAL void __launch_bounds__(256) lego_remap(const unsigned char* __restrict__ src,
                                                   unsigned char* __restrict__ dst,
                                                   long long src_stride, long long dst_stride) {
    const lego_e* s = reinterpret_cast<const lego_e*>(src) + (long long)blockIdx.y * src_stride;
    lego_e* d = reinterpret_cast<lego_e*>(dst) + (long long)blockIdx.y * dst_stride;
    for (long long f = (long long)blockIdx.x * blockDim.x + threadIdx.x; f < gen::N;
         f += (long long)gridDim.x * blockDim.x) {
        long long si;
        gen::src_of(f, si);
#if LEGO_MASKED
        d[f] = si >= 0 ? s[si] : (lego_e)0;
#else
        d[f] = s[si];
#endif
    }
}
#else
LEGO_GLOBAL void __launch_bounds__(256) lego_remap(const unsigned char* __restrict__ src,
                                                   unsigned char* __restrict__ dst,
                                                   long long src_stride, long long dst_stride) {
    const unsigned char* s = src + (long long)blockIdx.y * src_stride * LEGO_ELEM;
    unsigned char* d = dst + (long long)blockIdx.y * dst_stride * LEGO_ELEM;
    const long long nvec = gen::N / LEGO_VEC;
    const long long base = (long long)blockIdx.x * (blockDim.x * LEGO_UNROLL) + threadIdx.x;
    lego_v16 v[LEGO_UNROLL];
#pragma unroll
    for (int u = 0; u < LEGO_UNROLL; ++u) {
        const long long q = base + (long long)u * blockDim.x;
        if (q < nvec) v[u] = lego_gather_vec(s, q * LEGO_VEC);
    }
#pragma unroll
    for (int u = 0; u < LEGO_UNROLL; ++u) {
        const long long q = base + (long long)u * blockDim.x;
#if LEGO_ROUTED
        if (q < nvec) lego_st16(lego_route(dst, q * LEGO_VEC, LEGO_ELEM), v[u]);
#else
        if (q < nvec) lego_st16(d + q * 16, v[u]);
#endif
    }
}
#endif  // LEGO_SCALAR
#endif

// ---------------------------------------------------------------------------
#if LEGO_KIND == 2
// transpose of a digit permutation.  A warp owns a (4V) x (8V) tile: x runs
// along the dst-innermost digit (dst stride 1, src stride gen::SX), y along
// the src-innermost digit (src stride 1, dst stride gen::DY).  Lane (xg, yg)
// = (lane / 8, lane % 8) loads V rows x = xg*V + r of V elements along y
// (a 128-byte row segment per 8 lanes), transposes in registers and stores V
// rows y = yg*V + c of V elements along x.
#define LEGO_V (16 / LEGO_ELEM)
#ifndef LEGO_MINB
#define LEGO_MINB 1                   // min CTAs per SM for the register transpose (occupancy knob)
#endif

static __device__ __forceinline__ unsigned int lego_word(const lego_v16& v, int i) { return v.w[i]; }

#if LEGO_NARROW
// Interleave of a digit permutation with one innermost span below a 16-byte
// vector (lower.narrow_plan; AoS <-> SoA style).  NY = that span, NP = V/NY
// elements per chunk (a chunk is 16/NY bytes, contiguous on the other side).
// Mode 1: a thread loads one 16-byte source vector (P x-values x NY) and
// stores NY chunks, chunk y at gen::map(s + y); mode 2: a thread loads NY
// chunks, chunk x from gen::map(f + x), and stores one 16-byte vector.  The
// regrouping of the elements is register-only; every warp access is 32
// consecutive vectors (mode 1 loads, mode 2 stores) or 32 chunks at P-aligned
// positions that are contiguous across the lanes that share a run.
typedef lego_elem<LEGO_ELEM>::t lego_ne;
#define NY LEGO_NY
#define NP (LEGO_V / NY)
template <int B> struct lego_chunk;
template <> struct lego_chunk<1> { typedef unsigned char t; };
template <> struct lego_chunk<2> { typedef unsigned short t; };
template <> struct lego_chunk<4> { typedef unsigned int t; };
template <> struct lego_chunk<8> { typedef unsigned long long t; };
typedef lego_chunk<16 / NY>::t lego_ct;
LEGO_GLOBAL void __launch_bounds__(256) lego_remap(const unsigned char* __restrict__ src,
                                                   unsigned char* __restrict__ dst,
                                                   long long src_stride, long long dst_stride) {
    const unsigned char* s = src + (long long)blockIdx.y * src_stride * LEGO_ELEM;
    unsigned char* d = dst + (long long)blockIdx.y * dst_stride * LEGO_ELEM;
    const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= gen::N / LEGO_V) return;
    union { lego_v16 v; lego_ne e[LEGO_V]; } vec;
    union C { lego_ct c; lego_ne e[NP]; };
#if LEGO_NARROW == 1
    vec.v = lego_ld16(s + q * 16);
#pragma unroll
    for (int y = 0; y < NY; ++y) {
        long long pos;
        gen::map(q * LEGO_V + y, pos);
        C out;
#pragma unroll
        for (int p = 0; p < NP; ++p) out.e[p] = vec.e[p * NY + y];
        *reinterpret_cast<lego_ct*>(d + pos * LEGO_ELEM) = out.c;
    }
#else
#pragma unroll
    for (int x = 0; x < NY; ++x) {
        long long pos;
        gen::map(q * LEGO_V + x, pos);
        C in;
        in.c = __ldg(reinterpret_cast<const lego_ct*>(s + pos * LEGO_ELEM));
#pragma unroll
        for (int p = 0; p < NP; ++p) vec.e[p * NY + x] = in.e[p];
    }
    lego_st16(d + q * 16, vec.v);
#endif
}
#else

static __device__ __forceinline__ void lego_transpose(const lego_v16 (&in)[LEGO_V], lego_v16 (&out)[LEGO_V]) {
#if LEGO_ELEM == 4
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int r = 0; r < 4; ++r) out[c].w[r] = in[r].w[c];
#elif LEGO_ELEM == 2
#pragma unroll
    for (int c = 0; c < 8; ++c)
#pragma unroll
        for (int w = 0; w < 4; ++w)
            out[c].w[w] = __byte_perm(in[2 * w].w[c >> 1], in[2 * w + 1].w[c >> 1],
                                      (c & 1) ? 0x7632 : 0x5410);
#elif LEGO_ELEM == 8
    out[0].w[0] = in[0].w[0]; out[0].w[1] = in[0].w[1]; out[0].w[2] = in[1].w[0]; out[0].w[3] = in[1].w[1];
    out[1].w[0] = in[0].w[2]; out[1].w[1] = in[0].w[3]; out[1].w[2] = in[1].w[2]; out[1].w[3] = in[1].w[3];
#elif LEGO_ELEM == 1
#pragma unroll
    for (int c = 0; c < 16; ++c)
#pragma unroll
        for (int w = 0; w < 4; ++w) {
            const int sh = (c & 3) * 8;
            const unsigned int b0 = (in[4 * w + 0].w[c >> 2] >> sh) & 0xffu;
            const unsigned int b1 = (in[4 * w + 1].w[c >> 2] >> sh) & 0xffu;
            const unsigned int b2 = (in[4 * w + 2].w[c >> 2] >> sh) & 0xffu;
            const unsigned int b3 = (in[4 * w + 3].w[c >> 2] >> sh) & 0xffu;
            out[c].w[w] = b0 | (b1 << 8) | (b2 << 16) | (b3 << 24);
        }
#else
    out[0] = in[0];
#endif
}

#if LEGO_SMEM
// Variant with 128-byte segments on BOTH sides: a warp owns an (8V) x (8V)
// tile; lane (xg, c) = (lane / 8, lane % 8) loads two VxV blocks (x rows
// xg*V.. and (xg+4)*V..) along y chunk c, transposes them in registers and
// parks the x-vectors in shared memory as [y][x-chunk] 16-byte cells whose
// chunk index is XOR-swizzled by (y / V) % 8 (conflict-free both ways); the
// warp then writes 4 dst rows of 8 chunks (128 B each) per instruction.
LEGO_GLOBAL void __launch_bounds__(128) lego_remap(const unsigned char* __restrict__ src,
                                                   unsigned char* __restrict__ dst,
                                                   long long src_stride, long long dst_stride) {
    extern __shared__ lego_v16 lego_cells[];               // [warp][y][swizzled x-chunk]
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    lego_v16 (*cells)[8] = reinterpret_cast<lego_v16 (*)[8]>(lego_cells + warp * (8 * LEGO_V) * 8);
    const long long t = (long long)blockIdx.x * (blockDim.x >> 5) + warp;
    if (t >= gen::TILES) return;
    const unsigned char* s = src + (long long)blockIdx.y * src_stride * LEGO_ELEM;
    unsigned char* d = dst + (long long)blockIdx.y * dst_stride * LEGO_ELEM;
    long long f0, s0;
    gen::origin(t, f0, s0);
    const int c = lane & 7, xg = lane >> 3;
    lego_v16 rows[2][LEGO_V];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const unsigned char* sp =
            s + (s0 + (long long)((xg + 4 * h) * LEGO_V) * gen::SX + c * LEGO_V) * LEGO_ELEM;
#pragma unroll
        for (int r = 0; r < LEGO_V; ++r) rows[h][r] = lego_ld16(sp + (long long)r * gen::SX * LEGO_ELEM);
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        lego_v16 cols[LEGO_V];
        lego_transpose(rows[h], cols);
        const int xc = xg + 4 * h;                          // x-chunk of these vectors
#pragma unroll
        for (int m = 0; m < LEGO_V; ++m) {
            const int y = c * LEGO_V + m;
            cells[y][xc ^ (c & 7)] = cols[m];
        }
    }
    __syncwarp();
    // store: lanes 8q..8q+7 write dst row y (8 chunks = 128 bytes)
    const int k = lane & 7;
#pragma unroll
    for (int it = 0; it < 2 * LEGO_V; ++it) {
        const int y = it * 4 + (lane >> 3);
        const lego_v16 v = cells[y][k ^ ((y / LEGO_V) & 7)];
        lego_st16(d + (f0 + (long long)y * gen::DY + k * LEGO_V) * LEGO_ELEM, v);
    }
}
#elif LEGO_PERSIST
// Persistent variant: a fixed grid (a few CTAs per SM) whose warps stride
// over the warp tiles, loading tile t + stride while tile t is transposed and
// stored -- no CTA launch churn, and every lane always has a tile's worth of
// 16-byte loads in flight.
static __device__ __forceinline__ void lego_tile_load(const unsigned char* s, long long t, int xg, int yg,
                                                      long long& f0, lego_v16 (&rows)[LEGO_V]) {
    long long s0;
    gen::origin(t, f0, s0);
    const unsigned char* sp = s + (s0 + (long long)(xg * LEGO_V) * gen::SX + yg * LEGO_V) * LEGO_ELEM;
#pragma unroll
    for (int r = 0; r < LEGO_V; ++r) rows[r] = lego_ld16(sp + (long long)r * gen::SX * LEGO_ELEM);
}
static __device__ __forceinline__ void lego_tile_store(unsigned char* d, long long f0, int xg, int yg,
                                                       const lego_v16 (&rows)[LEGO_V]) {
    lego_v16 cols[LEGO_V];
    lego_transpose(rows, cols);
    unsigned char* dp = d + (f0 + (long long)(yg * LEGO_V) * gen::DY + xg * LEGO_V) * LEGO_ELEM;
#pragma unroll
    for (int c = 0; c < LEGO_V; ++c) lego_st16(dp + (long long)c * gen::DY * LEGO_ELEM, cols[c]);
}
LEGO_GLOBAL void __launch_bounds__(256, 2) lego_remap(const unsigned char* __restrict__ src,
                                                      unsigned char* __restrict__ dst,
                                                      long long src_stride, long long dst_stride) {
    const int lane = threadIdx.x & 31;
    const long long stride = (long long)gridDim.x * (blockDim.x >> 5);
    long long t = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (t >= gen::TILES) return;
    const unsigned char* s = src + (long long)blockIdx.y * src_stride * LEGO_ELEM;
    unsigned char* d = dst + (long long)blockIdx.y * dst_stride * LEGO_ELEM;
    const int yg = lane & 7, xg = lane >> 3;
    lego_v16 a[LEGO_V], b[LEGO_V];
    long long fa, fb;
    lego_tile_load(s, t, xg, yg, fa, a);
    for (;;) {
        const long long t1 = t + stride;
        if (t1 >= gen::TILES) { lego_tile_store(d, fa, xg, yg, a); return; }
        lego_tile_load(s, t1, xg, yg, fb, b);
        lego_tile_store(d, fa, xg, yg, a);
        const long long t2 = t1 + stride;
        if (t2 >= gen::TILES) { lego_tile_store(d, fb, xg, yg, b); return; }
        lego_tile_load(s, t2, xg, yg, fa, a);
        lego_tile_store(d, fb, xg, yg, b);
        t = t2;
    }
}
#else
#ifndef LEGO_TBLOCK
#define LEGO_TBLOCK 256
#endif
LEGO_GLOBAL void __launch_bounds__(LEGO_TBLOCK, LEGO_MINB) lego_remap(const unsigned char* __restrict__ src,
                                                   unsigned char* __restrict__ dst,
                                                   long long src_stride, long long dst_stride) {
    // LEGO_TPW warp tiles per warp: every tile's loads are issued before the
    // first transpose, so each lane keeps TPW*V 16-byte loads in flight
#ifndef LEGO_TPW
#define LEGO_TPW 1
#endif
    const int lane = threadIdx.x & 31;
    const long long t0 = ((long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * LEGO_TPW;
    if (t0 >= gen::TILES) return;
    const unsigned char* s = src + (long long)blockIdx.y * src_stride * LEGO_ELEM;
    unsigned char* d = dst + (long long)blockIdx.y * dst_stride * LEGO_ELEM;
#if LEGO_XMAJOR
    // 8 lanes along x (128-byte dst runs), 4 along y (64-byte src runs)
    const int xg = lane & 7, yg = lane >> 3;
#else
    // 8 lanes along y (128-byte src runs), 4 along x (64-byte dst runs)
    const int yg = lane & 7, xg = lane >> 3;
#endif
    long long f0[LEGO_TPW];
    lego_v16 rows[LEGO_TPW][LEGO_V];
#pragma unroll
    for (int u = 0; u < LEGO_TPW; ++u) {
        if (t0 + u >= gen::TILES) break;
        long long s0;
        gen::origin(t0 + u, f0[u], s0);
        const unsigned char* sp = s + (s0 + (long long)(xg * LEGO_V) * gen::SX + yg * LEGO_V) * LEGO_ELEM;
#pragma unroll
        for (int r = 0; r < LEGO_V; ++r) rows[u][r] = lego_ld16(sp + (long long)r * gen::SX * LEGO_ELEM);
    }
#pragma unroll
    for (int u = 0; u < LEGO_TPW; ++u) {
        if (t0 + u >= gen::TILES) break;
        lego_v16 cols[LEGO_V];
        lego_transpose(rows[u], cols);
#if LEGO_ROUTED
        const long long v0 = f0[u] + (long long)(yg * LEGO_V) * gen::DY + xg * LEGO_V;
#pragma unroll
        for (int c = 0; c < LEGO_V; ++c)
            lego_st16(lego_route(dst, v0 + (long long)c * gen::DY, LEGO_ELEM), cols[c]);
#else
        unsigned char* dp = d + (f0[u] + (long long)(yg * LEGO_V) * gen::DY + xg * LEGO_V) * LEGO_ELEM;
#pragma unroll
        for (int c = 0; c < LEGO_V; ++c) lego_st16(dp + (long long)c * gen::DY * LEGO_ELEM, cols[c]);
#endif
    }
}
#endif  // LEGO_SMEM
#endif  // LEGO_NARROW
#endif

// ---------------------------------------------------------------------------
#if LEGO_KIND == 3
// anti-diagonal band tiles.  The layout side is GroupBy([n,n]).OrderBy(GenP
// antidiag): its positions along one anti-diagonal t = i + j are consecutive
// in i, while row-major positions along one row are consecutive in j.  A CTA
// owns BR rows x BK anti-diagonals: the row-major side moves BR runs of BK
// consecutive elements (row i, columns t0-i ...), the layout side BK runs of
// BR consecutive elements (diagonal t, rows i0 ...), both coalesced, with
// the transpose done in padded shared memory.  gen::pos_of(x) is the
// generated antidiag apply (reference layout.py:564-570) evaluated once per
// run to find each diagonal run's base.  LEGO_DIR 0: row-major -> layout
// (scatter), 1: layout -> row-major (gather).
typedef lego_elem<LEGO_ELEM>::t lego_e;
#ifndef LEGO_BR
#define LEGO_BR 64
#endif
#ifndef LEGO_BK
#define LEGO_BK 64
#endif
#define BR LEGO_BR                                     // rows per band tile (multiple of 32)
#define BK LEGO_BK                                     // diagonals per band tile (multiple of 32, <= 256)
// 32-bit index arithmetic: the planner only selects this kernel when n*n < 2^31

#ifndef LEGO_BW
#define LEGO_BW 8                                      // warps per CTA
#endif
LEGO_GLOBAL void __launch_bounds__(32 * LEGO_BW) lego_remap(const unsigned char* __restrict__ src,
                                                   unsigned char* __restrict__ dst,
                                                   long long src_stride, long long dst_stride) {
    __shared__ lego_e tile[BR][BK + 1];
    __shared__ int run_base[BK];
    const int n = gen::NN;
    const lego_e* s = reinterpret_cast<const lego_e*>(src) + (long long)blockIdx.y * src_stride;
    lego_e* d = reinterpret_cast<lego_e*>(dst) + (long long)blockIdx.y * dst_stride;
#if LEGO_BAND_ORDER == 0
    // row-block major: consecutive CTAs walk the diagonals of one row block
    const int ri = blockIdx.x / gen::KBLOCKS;
    const int kk = blockIdx.x - ri * gen::KBLOCKS;
    const int i0 = ri * BR;
    const int t0 = (i0 / BK + kk) * BK;
#else
    // diagonal-block major: consecutive CTAs walk the row blocks of one band, so
    // the diagonal runs they write continue each other (L2 merges the seams)
    const int tb = blockIdx.x / (gen::NN / BR);
    const int i0 = (blockIdx.x - tb * (gen::NN / BR)) * BR;
    const int t0 = tb * BK;
    if (i0 > t0 + BK - 1) return;                      // rows below the band's reach
#endif
    if (t0 > i0 + BR - 1 + n - 1) return;             // band right of the matrix
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // base position of each diagonal's run: pos(i, t-i) = base_t + i
    for (int kk = threadIdx.x; kk < BK; kk += 32 * LEGO_BW) {
        const int t = t0 + kk;
        int iv = max(t - (n - 1), i0);
        int b = -1;
        if (t <= 2 * n - 2 && iv <= t && iv < i0 + BR) {
            long long p;
            gen::pos_of((long long)iv * n + (t - iv), p);
            b = (int)p - iv;
        }
        run_base[kk] = b;
    }
    constexpr int RPW = BR / LEGO_BW;                  // rows per warp
#if LEGO_DIR == 0
    {   // rows: BK consecutive elements of row i from column t0 - i; all loads first
        lego_e v[RPW][BK / 32];
#pragma unroll
        for (int q = 0; q < RPW; ++q) {
            const int i = i0 + warp + LEGO_BW * q;
            const int j0 = t0 - i;
            const lego_e* row = s + i * n;
#pragma unroll
            for (int h = 0; h < BK / 32; ++h) {
                const int j = j0 + 32 * h + lane;
                v[q][h] = ((unsigned)j < (unsigned)n) ? lego_lde(row + j) : (lego_e)0;
            }
        }
#pragma unroll
        for (int q = 0; q < RPW; ++q)
#pragma unroll
            for (int h = 0; h < BK / 32; ++h) tile[warp + LEGO_BW * q][32 * h + lane] = v[q][h];
    }
    __syncthreads();
    // diagonals: BR consecutive positions base_t + i
#pragma unroll
    for (int q = 0; q < BK / LEGO_BW; ++q) {
        const int k = warp + LEGO_BW * q;
        const int t = t0 + k;
        const int b = run_base[k];
        if (b < 0) continue;
#pragma unroll
        for (int h = 0; h < BR / 32; ++h) {
            const int i = i0 + 32 * h + lane;
            if ((unsigned)(t - i) < (unsigned)n) d[b + i] = tile[32 * h + lane][k];
        }
    }
#else
    __syncthreads();
    {
        lego_e v[BK / LEGO_BW][BR / 32];
#pragma unroll
        for (int q = 0; q < BK / LEGO_BW; ++q) {
            const int k = warp + LEGO_BW * q;
            const int t = t0 + k;
            const int b = run_base[k];
#pragma unroll
            for (int h = 0; h < BR / 32; ++h) {
                const int i = i0 + 32 * h + lane;
                v[q][h] = (b >= 0 && (unsigned)(t - i) < (unsigned)n) ? lego_lde(s + b + i) : (lego_e)0;
            }
        }
#pragma unroll
        for (int q = 0; q < BK / LEGO_BW; ++q)
#pragma unroll
            for (int h = 0; h < BR / 32; ++h) tile[32 * h + lane][warp + LEGO_BW * q] = v[q][h];
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < RPW; ++q) {
        const int i = i0 + warp + LEGO_BW * q;
        const int j0 = t0 - i;
        lego_e* row = d + i * n;
#pragma unroll
        for (int h = 0; h < BK / 32; ++h) {
            const int j = j0 + 32 * h + lane;
            if ((unsigned)j < (unsigned)n) row[j] = tile[warp + LEGO_BW * q][32 * h + lane];
        }
    }
#endif
}
#endif

// ---------------------------------------------------------------------------
#if LEGO_KIND == 4
// scatter: dst[apply(x)] = src[x] for a layout without an inverse (injective
// mode, reference layout.py:304-311, e.g. broadcast / even-map layouts).
// Each thread reads one 16-byte source vector (coalesced) and stores its
// elements at their generated positions; untouched positions keep the
// caller's initial values.
#define LEGO_VEC (16 / LEGO_ELEM)
typedef lego_elem<LEGO_ELEM>::t lego_e;

#if LEGO_SCALAR
LEGO_GLOBAL void __launch_bounds__(256) lego_remap(const unsigned char* __restrict__ src,
                                                   unsigned char* __restrict__ dst,
                                                   long long src_stride, long long dst_stride) {
    const lego_e* s = reinterpret_cast<const lego_e*>(src) + (long long)blockIdx.y * src_stride;
    lego_e* d = reinterpret_cast<lego_e*>(dst) + (long long)blockIdx.y * dst_stride;
    for (long long x = (long long)blockIdx.x * blockDim.x + threadIdx.x; x < gen::N;
         x += (long long)gridDim.x * blockDim.x) {
        long long p;
        gen::pos_of(x, p);
        if (p >= 0) d[p] = s[x];
    }
}
#else
LEGO_GLOBAL void __launch_bounds__(256) lego_remap(const unsigned char* __restrict__ src,
                                                   unsigned char* __restrict__ dst,
                                                   long long src_stride, long long dst_stride) {
    const unsigned char* s = src + (long long)blockIdx.y * src_stride * LEGO_ELEM;
    lego_e* d = reinterpret_cast<lego_e*>(dst + (long long)blockIdx.y * dst_stride * LEGO_ELEM);
    const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= gen::N / LEGO_VEC) return;
    union { lego_v16 v; lego_e e[LEGO_VEC]; } u;
    u.v = lego_ld16(s + q * 16);
#pragma unroll
    for (int k = 0; k < LEGO_VEC; ++k) {
        long long p;
        gen::pos_of(q * LEGO_VEC + k, p);
        if (p >= 0) d[p] = u.e[k];
    }
}
#endif  // LEGO_SCALAR

#if LEGO_FILL
// Fill mode: every destination position is written -- hit positions with
// their source element, the others with `fill` (raw element bits) -- so the
// destination needs no prior initialisation and no read-for-merge.
#if LEGO_FK > 0
// The planner proved apply(x) = FK*x + FC over the whole source (an affine
// injective layout, e.g. the even map FK = 2): source vector q (V elements)
// owns the destination window [FK*V*q + FC, FK*V*(q+1) + FC) of FK whole
// 16-byte vectors, which it assembles in registers and stores in full
// sectors; windows tile the destination.  Threads of q < ceil(FC/V) also
// fill the prefix [0, FC); the last window is clipped at N_DST.
#ifndef LEGO_FILL_UNROLL
#define LEGO_FILL_UNROLL 4
#endif
// The FK chunks of a lane's window are staged through shared memory so that
// every store instruction of a warp writes 32 consecutive 16-byte chunks
// (lane-interleaved windows would leave each instruction writing half
// sectors: measured 5.4 vs 6.x TB/s).
LEGO_GLOBAL void __launch_bounds__(256) lego_remap_fill(const unsigned char* __restrict__ src,
                                                        unsigned char* __restrict__ dst,
                                                        long long src_stride, long long dst_stride,
                                                        unsigned long long fill) {
    __shared__ lego_v16 stage[8][32 * LEGO_FK];
    const unsigned char* s = src + (long long)blockIdx.y * src_stride * LEGO_ELEM;
    lego_e* d = reinterpret_cast<lego_e*>(dst + (long long)blockIdx.y * dst_stride * LEGO_ELEM);
    const lego_e fv = (lego_e)fill;
    constexpr int U = LEGO_FILL_UNROLL;             // source vectors per thread, loads in flight together
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t * LEGO_VEC < LEGO_FC) {
#pragma unroll
        for (int k = 0; k < LEGO_VEC; ++k)
            if (t * LEGO_VEC + k < LEGO_FC) d[t * LEGO_VEC + k] = fv;
    }
    const long long nvec = gen::N / LEGO_VEC;
    // this warp's vectors: q0(u) + lane, q0(u) = (block * U + u) * 256 + 32 * warp
    union V { lego_v16 v; lego_e e[LEGO_VEC]; } in[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const long long q = ((long long)blockIdx.x * U + u) * 256 + 32 * warp + lane;
        if (q < nvec) in[u].v = lego_ld16(s + q * 16);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const long long q0 = ((long long)blockIdx.x * U + u) * 256 + 32 * warp;
        if (q0 >= nvec) break;
#pragma unroll
        for (int j = 0; j < LEGO_FK; ++j) {
            V out;
#pragma unroll
            for (int m = 0; m < LEGO_VEC; ++m) {
                const int w = j * LEGO_VEC + m;
                out.e[m] = (w % LEGO_FK == 0) ? in[u].e[w / LEGO_FK] : fv;
            }
            stage[warp][lane * LEGO_FK + j] = out.v;
        }
        __syncwarp();
        const long long w0 = (long long)LEGO_FK * LEGO_VEC * q0 + LEGO_FC;   // the warp's first window
        const long long lim = (long long)LEGO_FK * LEGO_VEC * nvec + LEGO_FC; // end of the windows
#pragma unroll
        for (int k = 0; k < LEGO_FK; ++k) {
            const int c = k * 32 + lane;
            const long long p = w0 + (long long)c * LEGO_VEC;
            V out;
            out.v = stage[warp][c];
            if (p + LEGO_VEC <= gen::N_DST && p + LEGO_VEC <= lim) {
                lego_st16(reinterpret_cast<unsigned char*>(d + p), out.v);
            } else {
#pragma unroll
                for (int m = 0; m < LEGO_VEC; ++m)
                    if (p + m < gen::N_DST && p + m < lim) d[p + m] = out.e[m];
            }
        }
        __syncwarp();
    }
}
#else
// General injective layouts: a vector fill of [0, N_DST) ahead of the scatter
// (lego_remap above), stream-ordered by the runtime.
LEGO_GLOBAL void __launch_bounds__(256) lego_remap_fill(const unsigned char* __restrict__ src,
                                                        unsigned char* __restrict__ dst,
                                                        long long src_stride, long long dst_stride,
                                                        unsigned long long fill) {
    (void)src;
    (void)src_stride;
    lego_e* d = reinterpret_cast<lego_e*>(dst + (long long)blockIdx.y * dst_stride * LEGO_ELEM);
    const lego_e fv = (lego_e)fill;
    const long long stride = (long long)gridDim.x * blockDim.x;
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const unsigned long long mis = (reinterpret_cast<unsigned long long>(d) & 15) / LEGO_ELEM;
    const long long head = mis ? (long long)(LEGO_VEC - mis) < gen::N_DST ? LEGO_VEC - mis : gen::N_DST : 0;
    for (long long k = t; k < head; k += stride) d[k] = fv;
    union { lego_v16 v; lego_e e[LEGO_VEC]; } u;
#pragma unroll
    for (int m = 0; m < LEGO_VEC; ++m) u.e[m] = fv;
    const long long nv = (gen::N_DST - head) / LEGO_VEC;
    for (long long k = t; k < nv; k += stride) lego_st16(reinterpret_cast<unsigned char*>(d + head + k * LEGO_VEC), u.v);
    for (long long k = head + nv * LEGO_VEC + t; k < gen::N_DST; k += stride) d[k] = fv;
}
#endif  // LEGO_FK
#endif  // LEGO_FILL
#endif

// ---------------------------------------------------------------------------
#if LEGO_KIND == 5
// box-staged gather (paper_2505_08091_b200/staging.py): the planner proved
// g(q*B + r) == base(q) + row(r)*SX + col(r), so destination block q (B
// consecutive elements) reads only the source box of R rows x C elements at
// stride SX starting at base(q), and reads every cell of it (so every cell is
// a valid source element: no bounds checks).  A CTA owns one block: coalesced (16-byte
// where aligned) loads of the box into shared memory (row pitch PITCH), then
// coalesced stores of the block, each element read from its box cell
// gen::TAB[r] = row(r)*PITCH + col(r) (a per-layout table, L1-resident).
//   LEGO_LVEC   box rows are whole 16-byte vectors at 16-byte stride (C*E and
//               SX*E multiples of 16); the start address is checked per CTA
//   LEGO_SVEC16 PITCH*E is a multiple of 16: box vectors stored whole
//   LEGO_VSTORE each thread stores V consecutive destination elements (one
//               16-byte store), else one element per lane
typedef lego_elem<LEGO_ELEM>::t lego_e;
#define LEGO_V (16 / LEGO_ELEM)
#ifndef LEGO_BT
#define LEGO_BT 256                                    // threads per CTA
#endif
struct alignas(sizeof(gen::tab_t) * LEGO_V) lego_tabv { gen::tab_t t[LEGO_V]; };

// store phase of the gather form: destination block from the staged box
static __device__ __forceinline__ void lego_box_store(const lego_e* box, lego_e* d, int tid) {
#if LEGO_VSTORE
    constexpr int NO = gen::B / LEGO_V;
#pragma unroll 4
    for (int k = tid; k < NO; k += LEGO_BT) {
        const lego_tabv tv = reinterpret_cast<const lego_tabv*>(gen::TAB)[k];
        union { lego_v16 v; lego_e e[LEGO_V]; } u;
#pragma unroll
        for (int e = 0; e < LEGO_V; ++e) u.e[e] = box[tv.t[e]];
        lego_st16(reinterpret_cast<unsigned char*>(d + (long long)k * LEGO_V), u.v);
    }
#else
#pragma unroll 8
    for (int r = tid; r < gen::B; r += LEGO_BT) d[r] = box[gen::TAB[r]];
#endif
}

#if LEGO_BULK
// TMA-fed persistent form (the planner proved base(q)*E, SX*E, C*E and
// PITCH*E are 16-byte multiples): each CTA walks blocks q = blockIdx.x,
// + gridDim.x, ...; warp 0 issues the next block's R box rows as 1-D bulk
// copies (cp.async.bulk, one per row, completing on an mbarrier with the
// byte count) into the other of two box buffers while all warps permute and
// store the current one.
static __device__ __forceinline__ void lego_mbar_wait(unsigned bar, unsigned parity) {
    asm volatile("{\n\t.reg .pred p;\n"
                 "LEGO_WAIT_%=:\n\t"
                 "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
                 "@!p bra LEGO_WAIT_%=;\n\t}" :: "r"(bar), "r"(parity) : "memory");
}
static __device__ __forceinline__ void lego_box_issue(const lego_e* s, long long q, unsigned box, unsigned bar,
                                                      int lane) {
    long long b0;
    gen::base_of(q, b0);
    constexpr unsigned ROWB = gen::C * LEGO_ELEM;
    if (lane == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                     :: "r"(bar), "r"((unsigned)(gen::R * ROWB)) : "memory");
    __syncwarp();
    for (int row = lane; row < gen::R; row += 32)
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     :: "r"(box + (unsigned)(row * gen::PITCH * LEGO_ELEM)),
                        "l"(s + b0 + (long long)row * gen::SX), "r"(ROWB), "r"(bar) : "memory");
}
LEGO_GLOBAL void __launch_bounds__(LEGO_BT) lego_remap(const unsigned char* __restrict__ src,
                                                       unsigned char* __restrict__ dst,
                                                       long long src_stride, long long dst_stride) {
    extern __shared__ __align__(128) unsigned char lego_smem[];
    constexpr unsigned BOXB = (gen::R * gen::PITCH * LEGO_ELEM + 127) / 128 * 128;
    const lego_e* s = reinterpret_cast<const lego_e*>(src) + (long long)blockIdx.y * src_stride;
    lego_e* d = reinterpret_cast<lego_e*>(dst) + (long long)blockIdx.y * dst_stride;
    const int tid = threadIdx.x;
    const long long nblk = gen::N / gen::B;
    const unsigned sbase = static_cast<unsigned>(__cvta_generic_to_shared(lego_smem));
    const unsigned bar = sbase + 2 * BOXB;
    if (((reinterpret_cast<unsigned long long>(s)) & 15) != 0) {
        // unaligned source (batch stride or pointer): per-thread element loads
        lego_e* box = reinterpret_cast<lego_e*>(lego_smem);
        for (long long q = blockIdx.x; q < nblk; q += gridDim.x) {
            long long b0;
            gen::base_of(q, b0);
            for (int k = tid; k < gen::R * gen::C; k += LEGO_BT) {
                const int row = k / gen::C, col = k - row * gen::C;
                box[row * gen::PITCH + col] = __ldg(s + b0 + (long long)row * gen::SX + col);
            }
            __syncthreads();
            lego_box_store(box, d + q * gen::B, tid);
            __syncthreads();
        }
        return;
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(bar) : "memory");
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(bar + 8) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    long long q = blockIdx.x;
    if (q >= nblk) return;
    if (tid < 32) lego_box_issue(s, q, sbase, bar, tid);
    for (int it = 0; q < nblk; q += gridDim.x, ++it) {
        const int buf = it & 1;
        const long long qn = q + gridDim.x;
        // buffer buf^1 was released by the barrier that ended the previous iteration
        if (qn < nblk && tid < 32) lego_box_issue(s, qn, sbase + (buf ^ 1) * BOXB, bar + 8 * (buf ^ 1), tid);
        lego_mbar_wait(bar + 8 * buf, (it >> 1) & 1);
        lego_box_store(reinterpret_cast<const lego_e*>(lego_smem + buf * BOXB), d + q * gen::B, tid);
        __syncthreads();
    }
}
#elif LEGO_SCATTER
// mirrored form: source block q (B consecutive elements) lands in the
// destination box at base(q) (R rows x C at stride SX): 16-byte loads of the
// block, scattered into the box cells gen::TAB[r], then box rows stored
// coalesced (16-byte where the row start is aligned).
LEGO_GLOBAL void __launch_bounds__(LEGO_BT) lego_remap(const unsigned char* __restrict__ src,
                                                       unsigned char* __restrict__ dst,
                                                       long long src_stride, long long dst_stride) {
    extern __shared__ __align__(16) unsigned char lego_smem[];
    lego_e* box = reinterpret_cast<lego_e*>(lego_smem);
    const long long q = blockIdx.x;
    const lego_e* s = reinterpret_cast<const lego_e*>(src) + (long long)blockIdx.y * src_stride + q * gen::B;
    lego_e* d = reinterpret_cast<lego_e*>(dst) + (long long)blockIdx.y * dst_stride;
    long long b0;
    gen::base_of(q, b0);
    const int tid = threadIdx.x;
    if ((reinterpret_cast<unsigned long long>(s) & 15) == 0) {
        constexpr int NV = gen::B / LEGO_V;
        constexpr int IT = (NV + LEGO_BT - 1) / LEGO_BT;
        lego_v16 v[IT];
#pragma unroll
        for (int it = 0; it < IT; ++it) {
            const int k = it * LEGO_BT + tid;
            if (k < NV) v[it] = lego_ld16(reinterpret_cast<const unsigned char*>(s + (long long)k * LEGO_V));
        }
#pragma unroll
        for (int it = 0; it < IT; ++it) {
            const int k = it * LEGO_BT + tid;
            if (k >= NV) break;
            const lego_tabv tv = reinterpret_cast<const lego_tabv*>(gen::TAB)[k];
            union { lego_v16 v; lego_e e[LEGO_V]; } u;
            u.v = v[it];
#pragma unroll
            for (int e = 0; e < LEGO_V; ++e) box[tv.t[e]] = u.e[e];
        }
    } else {
#pragma unroll 8
        for (int r = tid; r < gen::B; r += LEGO_BT) box[gen::TAB[r]] = __ldg(s + r);
    }
    __syncthreads();
    lego_e* db = d + b0;
#if LEGO_LVEC
    if ((reinterpret_cast<unsigned long long>(db) & 15) == 0) {
        constexpr int VPR = gen::C / LEGO_V;
        constexpr int NV = gen::R * VPR;
#pragma unroll 4
        for (int k = tid; k < NV; k += LEGO_BT) {
            const int row = k / VPR, cv = k - row * VPR;
#if LEGO_SVEC16
            const lego_v16 v = *reinterpret_cast<const lego_v16*>(box + row * gen::PITCH + cv * LEGO_V);
#else
            union { lego_v16 v; lego_e e[LEGO_V]; } u;
#pragma unroll
            for (int e = 0; e < LEGO_V; ++e) u.e[e] = box[row * gen::PITCH + cv * LEGO_V + e];
            const lego_v16 v = u.v;
#endif
            lego_st16(reinterpret_cast<unsigned char*>(db + (long long)row * gen::SX + cv * LEGO_V), v);
        }
    } else
#endif
    {
        constexpr int NC = gen::R * gen::C;
#pragma unroll 8
        for (int k = tid; k < NC; k += LEGO_BT) {
            const int row = k / gen::C, col = k - row * gen::C;
            db[(long long)row * gen::SX + col] = box[row * gen::PITCH + col];
        }
    }
}
#else
LEGO_GLOBAL void __launch_bounds__(LEGO_BT) lego_remap(const unsigned char* __restrict__ src,
                                                       unsigned char* __restrict__ dst,
                                                       long long src_stride, long long dst_stride) {
    extern __shared__ __align__(16) unsigned char lego_smem[];
    lego_e* box = reinterpret_cast<lego_e*>(lego_smem);
    const long long q = blockIdx.x;
    const lego_e* s = reinterpret_cast<const lego_e*>(src) + (long long)blockIdx.y * src_stride;
    lego_e* d = reinterpret_cast<lego_e*>(dst) + (long long)blockIdx.y * dst_stride + q * gen::B;
    long long b0;
    gen::base_of(q, b0);
    const int tid = threadIdx.x;
#if LEGO_LVEC
    const lego_e* sb = s + b0;
    if ((reinterpret_cast<unsigned long long>(sb) & 15) == 0) {
        constexpr int VPR = gen::C / LEGO_V;                 // vectors per box row
        constexpr int NV = gen::R * VPR;
        constexpr int IT = (NV + LEGO_BT - 1) / LEGO_BT;
        lego_v16 v[IT];
#pragma unroll
        for (int it = 0; it < IT; ++it) {
            const int k = it * LEGO_BT + tid;
            const int row = k / VPR, cv = k - row * VPR;
            if (k < NV)
                v[it] = lego_ld16(reinterpret_cast<const unsigned char*>(sb + (long long)row * gen::SX + cv * LEGO_V));
        }
#pragma unroll
        for (int it = 0; it < IT; ++it) {
            const int k = it * LEGO_BT + tid;
            const int row = k / VPR, cv = k - row * VPR;
            if (k >= NV) break;
#if LEGO_SVEC16
            *reinterpret_cast<lego_v16*>(box + row * gen::PITCH + cv * LEGO_V) = v[it];
#else
            union { lego_v16 v; lego_e e[LEGO_V]; } u;
            u.v = v[it];
#pragma unroll
            for (int e = 0; e < LEGO_V; ++e) box[row * gen::PITCH + cv * LEGO_V + e] = u.e[e];
#endif
        }
    } else
#endif
    {
        constexpr int NC = gen::R * gen::C;
        constexpr int IT = (NC + LEGO_BT - 1) / LEGO_BT;
#pragma unroll 8
        for (int it = 0; it < IT; ++it) {
            const int k = it * LEGO_BT + tid;
            if (k >= NC) break;
            const int row = k / gen::C, col = k - row * gen::C;
            const long long si = b0 + (long long)row * gen::SX + col;
            box[row * gen::PITCH + col] = __ldg(s + si);
        }
    }
    __syncthreads();
    lego_box_store(box, d, tid);
}
#endif  // LEGO_SCATTER
#endif
