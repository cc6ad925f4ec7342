// nw_kernels.cuh -- Needleman-Wunsch score matrix as a wavefront over LEGO
// tiles (BASELINE.json config 4b).  Kernel template shared by the static
// library kernel (wavefront.cu: column strips, row-major ring) and the
// programs generated from a user layout (kernels.nw_program: NVRTC, with a
// `namespace gen` of LEGO index functions in front of this file).
//
//   S[0][j] = -j*p,  S[i][0] = -i*p,
//   S[i][j] = max(S[i-1][j-1] + sim[i-1][j-1], S[i-1][j] - p, S[i][j-1] - p)
//
// Offset scores.  With S'[i][j] = S[i][j] + (i+j)*p the recurrence becomes
//   S'[i][j] = max(S'[i-1][j-1] + sim[i-1][j-1] + 2p, S'[i-1][j], S'[i][j-1])
// with all-zero borders: the left-to-right dependency chain is one integer
// max per cell (no subtract), and the conversion back to S happens in the
// store path, off the chain.  Exact whenever |p|*(2n+2) < 2^30 and the true
// scores fit in +-2^30 (checked on p; sim is the caller's contract).
//
// The layout (kernels.nw_layout; reference GroupBy/OrderBy semantics,
// pkg/src/lego/layout.py:206-334) over the cells of the padded n x n grid is
//   GroupBy([NR*H, NC*128]).OrderBy(RegP([NR,H,NC,128],[1,3,2,4])).OrderBy(T, I)
// i.e. position = T(a, b) * (H*128) + I(r, c) for cell (a*H + r, b*128 + c):
//  * T, the tile order, is the order in which CTAs claim tiles from an atomic
//    ticket: ticket t -> tile T^-1(t), generated as gen::tile_of.  The host
//    proves T is a topological order of the tile dependency graph (every
//    tile after its upper and left neighbours), so a persistent grid that
//    claims in ticket order never waits on an unclaimed tile;
//  * I, the cell order inside a tile, is the shared-memory order of the
//    tile's rows in the staging ring (the paper's LEGO-permuted NW buffer,
//    PAPER.md:1298-1301).  It must keep each row in its ring row and each
//    lane's 4-column group contiguous (one 16-byte vector); gen::slot(r, g)
//    gives the 16-byte slot of group g in tile row r.  The host proves both.
//
// Inside a tile (no host loop over diagonals, no grid sync), four warp roles
// per CTA, one per SM sub-partition:
//   warp 0  compute:  sweeps the tile in skewed 4x4 cell blocks -- lane j owns
//           columns 4j..4j+3 and at step s computes rows 4s - SKEW*(j+1) + q,
//           q = 0..3 (lane j runs SKEW rows behind lane j-1).  With SKEW = 1
//           row q of lane j takes its left value from row q-1 of lane j-1 in
//           the same step (one warp shuffle right after that row), so a
//           strip's 32 lanes are 32 rows apart instead of 32 steps (128 rows)
//           apart: the horizontal term of the wavefront's critical path
//           shrinks 4x.  Everything else is in registers or 16-byte shared
//           loads prefetched two steps ahead;
//   warp 1  producer: cp.async-stages sim, 32 rows x 128 columns per block,
//           into an 8-block ring (the compute warp overwrites each sim row
//           with its S' row in place);
//   warp 2  boundary: polls the left tile's published last column (32-bit
//           words in global memory, preset to a sentinel no offset score can
//           take) and hands it in row order, through a shared ring and a row
//           counter, to compute lane 0; in tiled mode it first fetches the
//           upper tile's published bottom row the same way;
//   warp 3  flusher:  converts finished blocks S' -> S and writes them out
//           as coalesced row segments.
// Roles synchronise through monotonic counters in shared memory (loaded /
// computed / flushed per 32-row block, ready per boundary row); the compute
// warp checks `loaded` once per block and `ready` every NW_GRP steps against
// prefetched values, so its step body has no barrier.
//
// Includer-provided switches:
//   NW_TILED      0: one tile per column strip (H = n, no top rows);
//                 1: tiles of H rows publish their bottom row for the tile below
//   NW_GEN_TILES  1: gen::tile_of(t, x) gives the row-major tile index x of ticket t
//   NW_GEN_SLOTS  1: gen::slot(r, g, s) gives the ring slot of lane group g in row r
#pragma once

#ifndef NW_TILED
#define NW_TILED 0
#endif
#ifndef NW_GEN_TILES
#define NW_GEN_TILES 0
#endif
#ifndef NW_GEN_SLOTS
#define NW_GEN_SLOTS 0
#endif
#ifndef NW_GLOBAL
#define NW_GLOBAL extern "C" __global__
#endif

namespace nwk {

typedef unsigned int u32;

constexpr int CPL = 4;                               // columns per lane
constexpr int STRIP = 32 * CPL;                      // columns per tile
constexpr int BLK = 32;                              // rows per block
#ifndef NW_RPS
#define NW_RPS 4                                     // rows per lane per step
#endif
constexpr int RPS = NW_RPS;
constexpr int STEPS = BLK / RPS;                     // compute steps per block
#ifndef NW_SKEW
#define NW_SKEW 1                                    // rows each lane runs behind its left neighbour (1, 2 or RPS)
#endif
constexpr int SKEW = NW_SKEW;
static_assert(SKEW >= 1 && SKEW <= RPS && RPS % SKEW == 0, "NW_SKEW must divide NW_RPS");
constexpr int LAG_BLKS = SKEW;                       // lane 31 runs 32*SKEW rows (SKEW blocks) behind the step's rows
constexpr int BLAG = LAG_BLKS + 1;                   // lane 31 completes block k before block k+BLAG starts
constexpr int DRAIN = LAG_BLKS;                      // extra blocks cover lane 31's lag
#ifndef NW_GRP
#define NW_GRP 2                                     // measured (n = 16384, SKEW 1): 1 step 912 us, 2 steps 882, 4 steps 897
#endif
constexpr int GRP = NW_GRP;                          // boundary readiness checked every GRP steps
#ifndef NW_NSLOT
#define NW_NSLOT (NW_SKEW == NW_RPS ? 12 : 8)        // lane 31 lags SKEW blocks: SKEW 1 needs fewer ring blocks
#endif
constexpr int NSLOT = NW_NSLOT;                      // ring blocks
constexpr int RING_ROWS = NSLOT * BLK;               // 256 (SKEW 1)
#ifndef NW_BND_ROWS
#define NW_BND_ROWS 256                              // boundary ring rows (must cover lane 31's lag: 512 for RPS 8)
#endif
constexpr int BND_ROWS = NW_BND_ROWS;               // boundary ring (rows)
constexpr int BND_GROUPS = BND_ROWS / BLK;
constexpr int ROW_BYTES = STRIP * 4;                 // 512
constexpr int RING_BYTES = RING_ROWS * ROW_BYTES;    // 128 KiB (SKEW 1)
constexpr int BND_BYTES = BND_ROWS * 4;
constexpr int MBAR_BYTES = NSLOT * 8;
constexpr int CTRL_BYTES = 64;
constexpr int TOP_BYTES = (STRIP + 4) * 4;           // upper tile's bottom row + the corner
constexpr int SMEM_BYTES = RING_BYTES + BND_BYTES + MBAR_BYTES + CTRL_BYTES + TOP_BYTES;
#define RING_POW2_PP ((NW_NSLOT & (NW_NSLOT - 1)) == 0)
#ifndef NW_PRODUCER_NS
#define NW_PRODUCER_NS 64                            // producer back-off when nothing landed or was issued
#endif
#ifndef NW_FLUSHER_NS
#define NW_FLUSHER_NS 64                             // flusher back-off while waiting for a computed block
#endif
#ifndef NW_POLL_NS
#define NW_POLL_NS 32                                // boundary poll back-off (measured: 32 ns 1068 us, 0 ns 1079 us)
#endif

// boundary words start as NW_EMPTY (|S'| < 2^30 never equals it)
constexpr int NW_EMPTY = (int)0x80808080;

#ifdef LEGO_NW_DEBUG
// event times (globaltimer ns, low 32 bits): g_nw_trace[(cta * 4 + role) * 2048 + idx]
__device__ unsigned g_nw_trace[148 * 4 * 2048];
__device__ __forceinline__ unsigned nw_now() {
    unsigned t;
    asm volatile("mov.u32 %0, %%globaltimer_lo;" : "=r"(t));
    return t;
}
#define NW_TRACE(role, idx) \
    do { if ((idx) < 2048) nwk::g_nw_trace[(blockIdx.x * 4 + (role)) * 2048 + (idx)] = nwk::nw_now(); } while (0)
#else
#define NW_TRACE(role, idx) ((void)0)
#endif

struct Ctrl {
    int tile;        // claimed ticket
    int loaded;      // sim blocks <= loaded have landed
    int computed;    // S' blocks <= computed are final
    int flushed;     // blocks <= flushed are written out (ring slot reusable)
    int ready;       // boundary rows < ready are in the shared ring
    int top;         // tiled mode: the upper tile's bottom row is in shared memory
};

// role counters in shared memory.  Publication is a release store at CTA
// scope (the guarded data was written before it, after a __syncwarp); the
// helper warps read counters with acquire loads.  The compute warp's hot
// loop polls `ready` / `loaded` with plain volatile loads: an acquire there
// costs 4 % of the kernel (1121 vs 1075 us at n = 16384), and the shared-
// memory accesses of one SM's warps are performed in issue order by its one
// shared-memory pipeline, which is what the pattern relies on.
__device__ __forceinline__ int ldv(const int* p) { return *reinterpret_cast<const volatile int*>(p); }
__device__ __forceinline__ int ldv_acq(const int* p) {
    int v;
    asm volatile("ld.acquire.cta.shared.b32 %0, [%1];" : "=r"(v)
                 : "r"((u32)__cvta_generic_to_shared(p)) : "memory");
    return v;
}
__device__ __forceinline__ void stv(int* p, int v) {
    asm volatile("st.release.cta.shared.b32 [%0], %1;" :: "r"((u32)__cvta_generic_to_shared(p)), "r"(v)
                 : "memory");
}

__device__ __forceinline__ void cp_async16(u32 dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async4(u32 dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" :: "r"(dst), "l"(src) : "memory");
}

__device__ __forceinline__ int ld_bnd(const int* p) {
    int w;
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(w) : "l"(p) : "memory");
    return w;
}
// system scope: a column band's edge polled by the next GPU over NVLink
__device__ __forceinline__ int ld_bnd_sys(const int* p) {
    int w;
    asm volatile("ld.relaxed.sys.global.b32 %0, [%1];" : "=r"(w) : "l"(p) : "memory");
    return w;
}
__device__ __forceinline__ int4 ld_bnd4(const int* p) {
    int4 w;
    asm volatile("ld.relaxed.gpu.global.v4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(w.x), "=r"(w.y), "=r"(w.z), "=r"(w.w) : "l"(p) : "memory");
    return w;
}

// ---------------------------------------------------------------------------
// LEGO maps: tile order and ring slots
// ---------------------------------------------------------------------------
// tile of ticket t (tiles row-major over NR x NC)
__device__ __forceinline__ void tile_of(long long t, int nc, int& a, int& b) {
#if NW_GEN_TILES
    long long x;
    gen::tile_of(t, x);
    a = (int)(x / nc);
    b = (int)(x - (long long)a * nc);
#else
    a = (int)(t / nc);
    b = (int)(t - (long long)a * nc);
#endif
}
// 16-byte slot of lane group g (columns 4g..4g+3) in tile row r
__device__ __forceinline__ int slot(int r, int g, int h) {
#if NW_GEN_SLOTS
    long long s;
    gen::slot((long long)min(max(r, 0), h - 1), (long long)g, s);
    return (int)s;
#else
    (void)r;
    (void)h;
    return g;
#endif
}

// compute-warp state: S' of the lane's 4 columns in its last finished row,
// the diagonal predecessor of its first column, the last-column values it
// sends right, the shuffled left values, and sim rows prefetched two steps ahead
#ifndef NW_ORDERED
#define NW_ORDERED 1             // shuffle, S' store and prefetch of each slot issued in order (volatile asm)
#endif
#ifndef NW_SHFL3
// lane 0's boundary as a third max operand (no select on the shuffle chain):
// strips 882.9 -> 864.5 us; tiled programs measured slower with it (128-row
// tiles 1584 -> 1623 us, 4096-row 1212 -> 1307), so strips only
#define NW_SHFL3 (!NW_TILED)
#endif
#ifndef NW_QFORM
#define NW_QFORM 1               // left-independent prefix maxima first: one max from the left value to x3
#endif
struct Lane {
    int h[CPL];
    int dprev;
    int send[RPS];
    int lin[RPS];            // lin[q]: the left neighbour's x3 of slot q (this step once slot q ran, else the last)
    int4 nx1[RPS], nx2[RPS];
    u32 o1[RPS], o2[RPS];    // ring byte offsets of the rows in nx1 / nx2 (the S' stores reuse them)
    u32 lanec;               // -SKEW*(lane+1)*ROW_BYTES + 16*lane: the lane's part of its ring offsets
    int bv[RPS];
};

__device__ __forceinline__ int max_opaque(int a, int b) {
    int r;
    asm("max.s32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}

template <int N>
__device__ __forceinline__ void ldsv(u32 a, int (&v)[N]);
template <>
__device__ __forceinline__ void ldsv<2>(u32 a, int (&v)[2]) {
    asm volatile("ld.volatile.shared.v2.b32 {%0,%1}, [%2];" : "=r"(v[0]), "=r"(v[1]) : "r"(a));
}
template <>
__device__ __forceinline__ void ldsv<8>(u32 a, int (&v)[8]) {
    asm volatile("ld.volatile.shared.v4.b32 {%0,%1,%2,%3}, [%8];\n\t"
                 "ld.volatile.shared.v4.b32 {%4,%5,%6,%7}, [%8+16];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(a));
}
template <>
__device__ __forceinline__ void ldsv<4>(u32 a, int (&v)[4]) {
    asm volatile("ld.volatile.shared.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
                 : "r"(a));
}

// predicated (branch-free) publication of RPS consecutive boundary words;
// SYS: system scope (column bands: the next GPU polls them)
template <bool SYS>
__device__ __forceinline__ void publish(int* p, int pred, const int (&v)[RPS]) {
#if NW_RPS == 4
    if (SYS) {
        asm volatile(
            "{\n\t.reg .pred q;\n\tsetp.ne.s32 q, %1, 0;\n\t"
            "@q st.relaxed.sys.global.v4.b32 [%0], {%2, %3, %4, %5};\n\t}"
            :: "l"(p), "r"(pred), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]) : "memory");
        return;
    }
#endif
#if NW_RPS == 8
    asm volatile(
        "{\n\t.reg .pred q;\n\tsetp.ne.s32 q, %1, 0;\n\t"
        "@q st.relaxed.gpu.global.v4.b32 [%0], {%2, %3, %4, %5};\n\t"
        "@q st.relaxed.gpu.global.v4.b32 [%0+16], {%6, %7, %8, %9};\n\t}"
        :: "l"(p), "r"(pred), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]),
           "r"(v[7]) : "memory");
#elif NW_RPS == 4
    asm volatile(
        "{\n\t.reg .pred q;\n\tsetp.ne.s32 q, %1, 0;\n\t"
        "@q st.relaxed.gpu.global.v4.b32 [%0], {%2, %3, %4, %5};\n\t}"
        :: "l"(p), "r"(pred), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]) : "memory");
#else
    asm volatile(
        "{\n\t.reg .pred q;\n\tsetp.ne.s32 q, %1, 0;\n\t"
        "@q st.relaxed.gpu.global.v2.b32 [%0], {%2, %3};\n\t}"
        :: "l"(p), "r"(pred), "r"(v[0]), "r"(v[1]) : "memory");
#endif
}
__device__ __forceinline__ void publish4(int* p, int pred, int x0, int x1, int x2, int x3) {
    asm volatile(
        "{\n\t.reg .pred q;\n\tsetp.ne.s32 q, %1, 0;\n\t"
        "@q st.relaxed.gpu.global.v4.b32 [%0], {%2, %3, %4, %5};\n\t}"
        :: "l"(p), "r"(pred), "r"(x0), "r"(x1), "r"(x2), "r"(x3) : "memory");
}

constexpr bool RING_POW2 = (RING_ROWS & (RING_ROWS - 1)) == 0;
__device__ __forceinline__ int ring_mod(int r) {
    if (RING_POW2) return r & (RING_ROWS - 1);
    int m = r % RING_ROWS;
    return m < 0 ? m + RING_ROWS : m;
}
// ring byte offset of lane group g's 16 bytes (columns 4g..4g+3) of tile row
// r: ring row r mod RING_ROWS, 16-byte slot slot(r, g)
__device__ __forceinline__ u32 cell_off(int r, int g, int h) {
    return (u32)(ring_mod(r) * ROW_BYTES + 16 * slot(r, g, h));
}

// Tile geometry shared by the roles.
struct Tile {
    int bm;          // matrix of the batch
    int a, b;        // tile row / column
    int row0, col0;  // first interior row / column
    int rows;        // interior rows in this tile
    int nblocks;     // 32-row blocks
    int* my_bnd;     // this tile column's right-column words, indexed by interior row
    int* top_in;     // tiled: the bottom row of the tile above (128 words), or null
    int* top_out;    // tiled: where this tile publishes its bottom row, or null
};

// one step of the compute warp: lane j computes the RPS x 4 block of tile rows
// r0 = RPS*s - SKEW*(j+1) .. r0+RPS-1, columns 4j..4j+3 of the tile.  Row q's
// left value is lane j-1's last column of its slot q-SKEW: from this step when
// q >= SKEW, else from the previous one.
template <bool GUARD, bool BAND>
__device__ __forceinline__ void nw_step(Lane& c, int s, int lane, unsigned char* ring, u32 bnd, int p2, const Tile& tl,
                                        int h, int* pub_row) {
    const int r0 = RPS * s - SKEW * (lane + 1);
    int4 cur[RPS];
    u32 so[RPS];
    int lb[RPS];
    const u32 ringa = static_cast<u32>(__cvta_generic_to_shared(ring));
#pragma unroll
    for (int q = 0; q < RPS; ++q) {
        cur[q] = c.nx1[q];
        so[q] = c.o1[q];
        c.nx1[q] = c.nx2[q];
        c.o1[q] = c.o2[q];
#if NW_GEN_SLOTS || !RING_POW2_PP
        c.o2[q] = cell_off(r0 + 2 * RPS + q, lane, h);
#else
        // (r mod RING_ROWS) * ROW_BYTES + 16*lane with one add and one mask:
        // 16*lane < ROW_BYTES and RING_BYTES divides 2^32
        c.o2[q] = ((u32)(s + 2) * (u32)(RPS * ROW_BYTES) + c.lanec + (u32)(q * ROW_BYTES)) & (u32)(RING_BYTES - 1);
#endif
#if !NW_ORDERED
#ifndef NW_ABL_NOLDS
        c.nx2[q] = *reinterpret_cast<const int4*>(ring + c.o2[q]);
#else
        c.nx2[q] = make_int4(q, lane, s, q ^ lane);
#endif
#endif
        lb[q] = c.bv[q];
    }
    ldsv<RPS>(bnd + (u32)(((RPS * (s + 1)) & (BND_ROWS - 1)) * 4), c.bv);   // next step's boundary
    int up0 = c.h[0], up1 = c.h[1], up2 = c.h[2], up3 = c.h[3];
    int d = c.dprev;
#pragma unroll
    for (int q = 0; q < RPS; ++q) {
#ifndef NW_ABL_LATESHFL
        const int left = lane == 0 ? lb[q] : c.lin[(q + RPS - SKEW) % RPS];
#else
        const int left = lane == 0 ? lb[q] : c.lin[q];   // ablation: last step's shuffle (wrong results)
#endif
        // lanes start SKEW rows apart; tiled: a lane stops at the tile's last
        // row, so its state ends on the bottom row published below the tile
        const bool live = !GUARD || (r0 + q >= 0 && (!NW_TILED || r0 + q < tl.rows));
#if NW_QFORM
        // prefix maxima of the row without its left value; x_c = max(Q_c, left).
        // The final maxima are opaque (asm) so the compiler cannot re-associate
        // them back into the 4-deep chain from `left`: left -> x3 is one op.
        const int q0 = max(cur[q].x + d + p2, up0);
        const int q1 = max(max(cur[q].y + up0 + p2, up1), q0);
        const int q2 = max(max(cur[q].z + up1 + p2, up2), q1);
        const int q3 = max(max(cur[q].w + up2 + p2, up3), q2);
#if NW_SHFL3
        // lane 0's left value enters through a third operand fixed before the
        // shuffle result arrives, so the shuffle chain has no select: lane 0's
        // own shuffle returns its previous row's x3 = up3 <= q3 (a column of S'
        // never decreases), which cannot change max(q3, boundary)
        const int sh = c.lin[(q + RPS - SKEW) % RPS];
        const int bvm = lane == 0 ? lb[q] : (-2147483647 - 1);
        int x3;
        asm("max.s32 %0, %1, %2;\n\tmax.s32 %0, %0, %3;" : "=&r"(x3) : "r"(q3), "r"(bvm), "r"(sh));
        const int x3s = GUARD && !live ? up3 : x3;   // a dead slot shuffles a value its right lane may take as up3
#else
        const int x3 = max_opaque(q3, left);
        const int x3s = x3;
#endif
#if NW_ORDERED
        asm volatile("shfl.sync.up.b32 %0, %1, 1, 0, 0xffffffff;" : "=r"(c.lin[q]) : "r"(x3s));
#else
        c.lin[q] = __shfl_up_sync(0xffffffffu, x3s, 1);
#endif
        const int x0 = max_opaque(q0, left);
        const int x1 = max_opaque(q1, left);
        const int x2 = max_opaque(q2, left);
#else
        const int x0 = max(max(cur[q].x + d + p2, up0), left);
        const int x1 = max(max(cur[q].y + up0 + p2, up1), x0);
        const int x2 = max(max(cur[q].z + up1 + p2, up2), x1);
        const int x3 = max(max(cur[q].w + up2 + p2, up3), x2);
        c.lin[q] = __shfl_up_sync(0xffffffffu, x3, 1);
#endif
#if NW_ORDERED
        // the slot's shared-memory traffic right behind its shuffle, in
        // program order (volatile asm): the next slot's shuffle does not queue
        // behind a burst of 128-bit stores and loads
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %5, 0;\n\t"
                     "@p st.shared.v4.b32 [%0], {%1, %2, %3, %4};\n\t}"
                     :: "r"(ringa + so[q]), "r"(x0), "r"(x1), "r"(x2), "r"(x3), "r"((u32)live) : "memory");
        asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(c.nx2[q].x), "=r"(c.nx2[q].y), "=r"(c.nx2[q].z), "=r"(c.nx2[q].w)
                     : "r"(ringa + c.o2[q]) : "memory");
#elif !defined(NW_ABL_NOSTS)
        if (live) *reinterpret_cast<int4*>(ring + so[q]) = make_int4(x0, x1, x2, x3);   // S' replaces sim in place
#endif
        up0 = live ? x0 : up0;
        up1 = live ? x1 : up1;
        up2 = live ? x2 : up2;
        up3 = live ? x3 : up3;
        d = live ? left : d;
        c.send[q] = x3;
    }
    c.h[0] = up0;
    c.h[1] = up1;
    c.h[2] = up2;
    c.h[3] = up3;
    c.dprev = d;
    // the tile's last column goes to the right neighbour (lane 31: r0 is a
    // multiple of 4, so its RPS rows are all live or all not)
    const int pub = (lane == 31) & (r0 >= 0) & (r0 < tl.rows);
#ifndef NW_ABL_NOPUB
    publish<BAND>(pub_row, pub, c.send);
#endif
#ifdef LEGO_NW_DEBUG
    if (pub && r0 < 512) NW_TRACE(3, 1536 + r0 / 4);   // lane 31 published rows r0..r0+3
#endif
}

// one block of STEPS steps (lane 0's rows 32k - SKEW ..); boundary readiness is
// checked every GRP steps against a counter value prefetched GRP steps earlier
template <bool GUARD, bool BAND>
__device__ __forceinline__ void nw_block(Lane& c, int k, int lane, unsigned char* ring, u32 bnd, int p2, const Tile& tl,
                                         int h, int& rd, const int* ready, int rows_total) {
    int* pub_blk = tl.my_bnd + tl.row0 + k * BLK - 32 * SKEW;  // lane 31's rows of step u: + RPS*u
#pragma unroll
    for (int u = 0; u < STEPS; ++u) {
        const int s = k * STEPS + u;
        if (u % GRP == 0) {                             // rows used (and prefetched) through step s + GRP
            const int need = min(RPS * (s + GRP + 1), rows_total);   // the helper stops at rows_total
            while (rd < need) rd = ldv(ready);
            rd = ldv(ready);
            if (lane == 0 && s < 512) NW_TRACE(0, 1536 + s);   // readiness check passed
        }
        nw_step<GUARD, BAND>(c, s, lane, ring, bnd, p2, tl, h, pub_blk + RPS * u);
    }
}

// Kernel body.  Tiles: NR x NC per matrix, H rows x 128 columns each
// (NR = 1, H = n in strip mode); total = batch * NR * NC tickets.
// bnd_g: per (matrix, tile column) n_pad words (the column's right edge,
// by interior row); top_g (tiled): per (matrix, tile) 128 words (the bottom
// row of the tile above it).  Both preset to NW_EMPTY by the launcher.
// BAND (strip mode): this launch owns strips strip_base .. strip_base +
// nc_band - 1 of the matrices' nc; bnd_g holds only those strips' edge
// columns, and the first one's left edge is read from left_ext (the previous
// band's last edge column, possibly another GPU's memory; matrix bm at
// left_ext + bm * left_bstride)
template <bool BAND = false>
__device__ __forceinline__ void nw_tiles_body(const int* __restrict__ sim, int* __restrict__ score, int n, int p,
                                              int H, int nr, int nc, int total, int* __restrict__ ticket,
                                              int* __restrict__ bnd_g, int* __restrict__ top_g,
                                              int strip_base = 0, int nc_band = 0, const int* left_ext = nullptr,
                                              long long left_bstride = 0) {
    extern __shared__ __align__(16) unsigned char smem[];
    int* ring_gen = reinterpret_cast<int*>(smem);
    Ctrl* ctrl = reinterpret_cast<Ctrl*>(smem + RING_BYTES + BND_BYTES + MBAR_BYTES);
    int* top_s = reinterpret_cast<int*>(smem + RING_BYTES + BND_BYTES + MBAR_BYTES + CTRL_BYTES);
    const u32 ring = static_cast<u32>(__cvta_generic_to_shared(smem));
    const u32 bnd = ring + RING_BYTES;
    const u32 mbar = bnd + BND_BYTES;
    int gblk = 0;                                    // producer: blocks issued in earlier tiles
    if (threadIdx.x < NSLOT)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 32;" :: "r"(mbar + 8u * threadIdx.x) : "memory");
    const int lane = threadIdx.x & 31;
    const int warp = __shfl_sync(0xffffffffu, (int)threadIdx.x >> 5, 0);   // warp-uniform role
    const int n_pad = (n + BLK - 1) / BLK * BLK;
    const int ncb = BAND ? nc_band : nc;             // tile columns this launch owns
    const int tiles_per_matrix = nr * ncb;

    for (;;) {
        if (threadIdx.x == 0) {
            ctrl->tile = atomicAdd(ticket, 1);
            ctrl->loaded = ctrl->computed = ctrl->flushed = -1;
            ctrl->ready = 0;
            ctrl->top = 0;
        }
        __syncthreads();
        const int t = ctrl->tile;
        if (t >= total) return;
#ifdef LEGO_NW_DEBUG
        if (threadIdx.x == 0) g_nw_trace[(blockIdx.x * 4 + 3) * 2048 + 2047] = (unsigned)t + 1;   // tile of this CTA
#endif
        Tile tl;
        tl.bm = t / tiles_per_matrix;
        tile_of(t - tl.bm * tiles_per_matrix, ncb, tl.a, tl.b);
        if (BAND) tl.b += strip_base;
        tl.row0 = tl.a * H;
        tl.col0 = tl.b * STRIP;
        tl.rows = min(H, n - tl.row0);
        tl.nblocks = (tl.rows + BLK - 1) / BLK;
        tl.my_bnd = bnd_g + (long long)(tl.bm * ncb + (tl.b - (BAND ? strip_base : 0))) * n_pad;
#if NW_TILED
        {
            const long long tid = (long long)tl.bm * tiles_per_matrix + (long long)tl.a * nc + tl.b;
            tl.top_in = tl.a > 0 ? top_g + tid * STRIP : nullptr;
            tl.top_out = tl.a + 1 < nr ? top_g + (tid + nc) * STRIP : nullptr;
        }
#else
        tl.top_in = tl.top_out = nullptr;
        (void)top_s;
#endif
        const int rows_total = (tl.nblocks + DRAIN) * BLK;

        if (warp == 0) {
            // ---------------- compute ----------------
            Lane c;
#pragma unroll
            for (int q = 0; q < CPL; ++q) c.h[q] = 0;
#pragma unroll
            for (int q = 0; q < RPS; ++q) c.send[q] = c.lin[q] = 0;
            c.dprev = 0;
#if NW_TILED
            if (tl.top_in) {                            // S' of the row above the tile
                while (ldv_acq(&ctrl->top) == 0) {}
#pragma unroll
                for (int q = 0; q < CPL; ++q) c.h[q] = top_s[CPL * lane + q];
                c.dprev = lane == 0 ? top_s[STRIP] : top_s[CPL * lane - 1];
            }
#endif
            const int p2 = 2 * p;
            c.lanec = (u32)(16 * lane) - (u32)(SKEW * (lane + 1) * ROW_BYTES);
            int pl = ldv(&ctrl->loaded);
            int rd = ldv(&ctrl->ready);
            for (int k = 0; k < tl.nblocks + DRAIN; ++k) {
                if (lane == 0) NW_TRACE(0, k);
                if (k >= BLAG) {                        // lane 31 has finished block k - BLAG
                    __syncwarp();
                    if (lane == 0) stv(&ctrl->computed, k - BLAG);
                }
                // the last steps of block k prefetch block k+1's first rows: need both
                const int need_blk = min(k + 1, tl.nblocks + DRAIN - 1);
                while (pl < need_blk) pl = ldv(&ctrl->loaded);
                if (lane == 0) NW_TRACE(0, 1024 + k);      // operands in
                if (k == 0) {                           // operands of the first two steps
                    while (rd < RPS) rd = ldv(&ctrl->ready);
#pragma unroll
                    for (int q = 0; q < RPS; ++q) {
                        c.o1[q] = cell_off(q - SKEW * (lane + 1), lane, H);
                        c.o2[q] = cell_off(RPS + q - SKEW * (lane + 1), lane, H);
                        c.nx1[q] = *reinterpret_cast<const int4*>(smem + c.o1[q]);
                        c.nx2[q] = *reinterpret_cast<const int4*>(smem + c.o2[q]);
                    }
                    ldsv<RPS>(bnd, c.bv);
                }
                pl = ldv(&ctrl->loaded);                // prefetch for the next block
                if (k < LAG_BLKS || (NW_TILED && k + 1 >= tl.nblocks))   // lane 31's first rows are negative; tiled: rows past the tile
                    nw_block<true, BAND>(c, k, lane, smem, bnd, p2, tl, H, rd, &ctrl->ready, rows_total);
                else
                    nw_block<false, BAND>(c, k, lane, smem, bnd, p2, tl, H, rd, &ctrl->ready, rows_total);
            }
#if NW_TILED
            // the tile's last row (each lane's state stopped there) goes to the tile below
            publish4(tl.top_out + 4 * lane, tl.top_out != nullptr, c.h[0], c.h[1], c.h[2], c.h[3]);
#endif
            __syncwarp();
            if (lane == 0) stv(&ctrl->computed, tl.nblocks + DRAIN - 1);
        } else if (warp == 1) {
            // ---------------- producer: sim blocks -> ring ----------------
            // Issues block k once its ring slot is flushed; each block's
            // copies arrive on a per-slot mbarrier, polled without blocking so
            // `loaded` is published as soon as a block lands.
            const int* simb = sim + (long long)tl.bm * n * n + (long long)tl.row0 * n;
            const bool vec = (n & 3) == 0;
            const int total_blocks = tl.nblocks + DRAIN;
            int issued = 0, landed = 0;
            while (landed < total_blocks) {
                bool progress = false;
                if (issued < total_blocks && (issued < NSLOT || ldv_acq(&ctrl->flushed) >= issued - NSLOT)) {
                    const int k = issued;
                    const u32 mb = mbar + 8u * (u32)((gblk + k) % NSLOT);
#ifndef NW_ABL_NOSIM
                    if (k < tl.nblocks) {
#else
                    if (false) {                        // ablation: no sim staging (wrong results)
#endif
                        const int rows = min(BLK, tl.rows - k * BLK);
                        const u32 blk = ring + (u32)((k % NSLOT) * BLK * ROW_BYTES);
                        if (vec) {
                            const bool ok = tl.col0 + CPL * lane < n;
#ifndef NW_ABL_SIMCACHED
                            const int* src = simb + (long long)k * BLK * n + tl.col0 + CPL * lane;
#else
                            const int* src = simb + tl.col0 + CPL * lane;   // ablation: L2-resident rows (wrong results)
#endif
#pragma unroll 8
                            for (int r = 0; r < rows; ++r) {
                                if (ok) cp_async16(blk + (u32)(r * ROW_BYTES + 16 * slot(k * BLK + r, lane, H)), src);
                                src += n;
                            }
                        } else {
                            const int* src = simb + (long long)k * BLK * n + tl.col0 + lane;
                            for (int r = 0; r < rows; ++r) {
#pragma unroll
                                for (int q = 0; q < CPL; ++q) {
                                    const int col = 32 * q + lane;
                                    if (tl.col0 + col < n)
                                        cp_async4(blk + (u32)(r * ROW_BYTES + 16 * slot(k * BLK + r, col >> 2, H)
                                                              + 4 * (col & 3)), src + 32 * q);
                                }
                                src += n;
                            }
                        }
                        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" :: "r"(mb) : "memory");
                        if (lane == 0) NW_TRACE(1, 1024 + k);  // block issued
                    } else {
                        asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}"
                                     :: "r"(mb) : "memory");
                    }
                    ++issued;
                    progress = true;
                }
                if (landed < issued) {
                    const int g = gblk + landed;
                    u32 ok;
                    asm volatile("{\n\t.reg .pred p;\n\t"
                                 "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                                 "selp.u32 %0, 1, 0, p;\n\t}"
                                 : "=r"(ok) : "r"(mbar + 8u * (u32)(g % NSLOT)), "r"((g / NSLOT) & 1)
                                 : "memory");
                    if (__all_sync(0xffffffffu, ok)) {
                        if (lane == 0) {
                            stv(&ctrl->loaded, landed);
                            NW_TRACE(1, landed);
                        }
                        ++landed;
                        progress = true;
                    }
                }
                if (!progress) __nanosleep(NW_PRODUCER_NS);
            }
            gblk += total_blocks;
        } else if (warp == 2) {
            // ---------------- boundary: neighbours' edges -> shared memory ----------------
#if NW_TILED
            if (tl.top_in) {
                // the upper tile's bottom row (lane l: columns 4l..4l+3) and the
                // corner S'[row0-1][col0-1] (the left column's word, or the border)
                int4 v = ld_bnd4(tl.top_in + CPL * lane);
                while (v.x == NW_EMPTY || v.y == NW_EMPTY || v.z == NW_EMPTY || v.w == NW_EMPTY) {
                    __nanosleep(NW_POLL_NS);
                    v = ld_bnd4(tl.top_in + CPL * lane);
                }
                top_s[CPL * lane + 0] = v.x;
                top_s[CPL * lane + 1] = v.y;
                top_s[CPL * lane + 2] = v.z;
                top_s[CPL * lane + 3] = v.w;
                if (lane == 0) {
                    int corner = 0;
                    if (tl.b > 0) {
                        const int* cp = tl.my_bnd - n_pad + tl.row0 - 1;
                        corner = ld_bnd(cp);
                        while (corner == NW_EMPTY) {
                            __nanosleep(NW_POLL_NS);
                            corner = ld_bnd(cp);
                        }
                    }
                    top_s[STRIP] = corner;
                }
                __syncwarp();
                if (lane == 0) stv(&ctrl->top, 1);
            }
#endif
            // Lane l polls row 32m + l of the left column; rows are handed to
            // the compute warp in order through ctrl->ready as soon as a
            // prefix of the group is in.  Row r sits at ring index r + SKEW,
            // so lane 0's rows 4s - SKEW .. 4s - SKEW + 3 are one aligned
            // 16-byte load.
            const bool ext = BAND && tl.b == strip_base && left_ext != nullptr;   // the previous band's edge
            const int* left = ext ? left_ext + tl.bm * left_bstride + tl.row0 : tl.my_bnd - n_pad + tl.row0;
            const int groups = tl.nblocks + DRAIN;
            for (int m = 0; m < groups; ++m) {
                const int r = m * BLK + lane;
                if (m >= BND_GROUPS) {
                    while (ldv_acq(&ctrl->computed) < m - BND_GROUPS) __nanosleep(128);
                }
                int v = 0;                              // S'[r+1][0] = 0 on the matrix edge
                bool ok = true;
                if (tl.b > 0 && r < tl.rows) {
                    v = ext ? ld_bnd_sys(left + r) : ld_bnd(left + r);
                    ok = v != NW_EMPTY;
                }
                bool written = false;
                int told = 0;
                for (;;) {
                    const unsigned ball = __ballot_sync(0xffffffffu, ok);
                    const int tt = ball == 0xffffffffu ? 32 : __ffs(~ball) - 1;   // ready prefix
                    if (ok && !written && lane < tt) {
                        asm volatile("st.shared.b32 [%0], %1;" :: "r"(bnd + (u32)(((r + SKEW) & (BND_ROWS - 1)) * 4)),
                                     "r"(v) : "memory");
                        written = true;
                    }
                    if (tt > told) {
                        __syncwarp();
                        if (lane == 0) stv(&ctrl->ready, m * BLK + tt);
#ifdef LEGO_NW_DEBUG
                        if (lane == 0 && m * BLK + tt <= 512)      // time row (m*BLK + tt - 1) became ready
                            for (int x = m * BLK + told; x < m * BLK + tt; ++x) NW_TRACE(2, 1024 + x);
#endif
                        told = tt;
                    }
                    if (tt == 32) break;
                    if (NW_POLL_NS) __nanosleep(NW_POLL_NS);
                    if (!ok) {
                        v = ext ? ld_bnd_sys(left + r) : ld_bnd(left + r);
                        ok = v != NW_EMPTY;
                    }
                }
                if (lane == 31) NW_TRACE(2, m);
            }
        } else {
            // ---------------- flusher: S' -> S, coalesced row segments ----------------
            int* sc = score + (long long)tl.bm * ((long long)n + 1) * ((long long)n + 1);
            const long long ld = (long long)n + 1;
            bool ok[CPL];
#pragma unroll
            for (int q = 0; q < CPL; ++q) ok[q] = tl.col0 + 32 * q + lane < n;
            for (int k = 0; k < tl.nblocks; ++k) {
                while (ldv_acq(&ctrl->computed) < k) __nanosleep(NW_FLUSHER_NS);
                if (lane == 0) NW_TRACE(3, 1024 + k);      // block computed: flush starts
                const int rows = min(BLK, tl.rows - k * BLK);
#ifdef NW_ABL_NOFLUSH
                if (rows > 0) { __syncwarp(); if (lane == 0) stv(&ctrl->flushed, k); continue; }   // ablation: no output
#endif
                const int* src = ring_gen + (k % NSLOT) * BLK * STRIP;
                int* dst = sc + (long long)(tl.row0 + k * BLK + 1) * ld + tl.col0 + 1 + lane;
                int off = (tl.row0 + k * BLK + tl.col0 + lane + 2) * p;   // (i + j) * p of column lane, row k*BLK
#if NW_GEN_SLOTS
                // cell (r, 32q + lane) sits at slot(r, (32q + lane) / 4) * 4 + lane % 4 of its ring row
                if (rows == BLK && tl.col0 + STRIP <= n) {
                    // full block: 16 rows of loads in flight before their stores
#pragma unroll
                    for (int hh = 0; hh < 2; ++hh) {
                        int v[16][CPL];
#pragma unroll
                        for (int r = 0; r < 16; ++r)
#pragma unroll
                            for (int q = 0; q < CPL; ++q)
                                v[r][q] = src[(16 * hh + r) * STRIP
                                              + 4 * slot(k * BLK + 16 * hh + r, 8 * q + (lane >> 2), H) + (lane & 3)];
#pragma unroll
                        for (int r = 0; r < 16; ++r) {
                            int* d = dst + (16 * hh + r) * ld;
                            const int o = off + (16 * hh + r) * p;
#pragma unroll
                            for (int q = 0; q < CPL; ++q) d[32 * q] = v[r][q] - (o + 32 * q * p);
                        }
                    }
                } else {
#pragma unroll 2
                    for (int r = 0; r < rows; ++r) {
#pragma unroll
                        for (int q = 0; q < CPL; ++q)
                            if (ok[q])
                                dst[32 * q] = src[r * STRIP + 4 * slot(k * BLK + r, 8 * q + (lane >> 2), H) + (lane & 3)]
                                              - (off + 32 * q * p);
                        dst += ld;
                        off += p;
                    }
                }
#else
                if (rows == BLK && tl.col0 + STRIP <= n) {
                    // full block: 16 rows of loads in flight before their stores
#pragma unroll
                    for (int hh = 0; hh < 2; ++hh) {
                        int v[16][CPL];
#pragma unroll
                        for (int r = 0; r < 16; ++r)
#pragma unroll
                            for (int q = 0; q < CPL; ++q) v[r][q] = src[(16 * hh + r) * STRIP + 32 * q + lane];
#pragma unroll
                        for (int r = 0; r < 16; ++r) {
                            int* d = dst + (16 * hh + r) * ld;
                            const int o = off + (16 * hh + r) * p;
#pragma unroll
                            for (int q = 0; q < CPL; ++q) d[32 * q] = v[r][q] - (o + 32 * q * p);
                        }
                    }
                } else {
                    src += lane;
#pragma unroll 4
                    for (int r = 0; r < rows; ++r) {
#pragma unroll
                        for (int q = 0; q < CPL; ++q)
                            if (ok[q]) dst[32 * q] = src[32 * q] - (off + 32 * q * p);
                        dst += ld;
                        src += STRIP;
                        off += p;
                    }
                }
#endif
                __syncwarp();
                if (lane == 0) { stv(&ctrl->flushed, k); NW_TRACE(3, k); }
            }
        }
        __syncthreads();
    }
}

__device__ __forceinline__ void nw_borders_body(int* __restrict__ score, long long n, int p, long long batch) {
    const long long w = n + 1;
    const long long total = batch * w;
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < total;
         k += (long long)gridDim.x * blockDim.x) {
        const long long b = k / w, x = k - b * w;
        int* s = score + b * w * w;
        s[x] = (int)(-x * p);          // row 0
        s[x * w] = (int)(-x * p);      // column 0
    }
}

}  // namespace nwk

// launch entry points (extern "C" in generated programs: cuModuleGetFunction names)
NW_GLOBAL void __launch_bounds__(128, 1)
lego_nw_tiles(const int* __restrict__ sim, int* __restrict__ score, int n, int p, int H, int nr, int nc, int total,
              int* __restrict__ ticket, int* __restrict__ bnd_g, int* __restrict__ top_g) {
    nwk::nw_tiles_body(sim, score, n, p, H, nr, nc, total, ticket, bnd_g, top_g);
}

#ifdef NW_BAND_ENTRY
// column band of strip-mode tiles (multi-GPU single alignment, shard.py)
NW_GLOBAL void __launch_bounds__(128, 1)
lego_nw_band(const int* __restrict__ sim, int* __restrict__ score, int n, int p, int nc, int total,
             int* __restrict__ ticket, int* __restrict__ bnd_g, int strip_base, int nc_band,
             const int* __restrict__ left_ext, long long left_bstride) {
    nwk::nw_tiles_body<true>(sim, score, n, p, n, 1, nc, total, ticket, bnd_g, nullptr, strip_base, nc_band,
                             left_ext, left_bstride);
}
#endif

NW_GLOBAL void lego_nw_borders(int* __restrict__ score, long long n, int p, long long batch) {
    nwk::nw_borders_body(score, n, p, batch);
}
