/*
 * lego_b200.h -- C ABI of the B200 execution backend for the LEGO layout
 * language (arXiv 2505.08091).
 *
 * The reference package (/root/reference/pkg/src/lego) is pure Python and
 * has no FFI; its hot path is the per-element scalar call
 *     GroupBy.apply(idx)  (layout.py:313-318)   logical index -> position
 *     GroupBy.inv(flat)   (layout.py:320-328)   position -> logical index
 * (ExpandBy.apply/inv, layout.py:383-400, for partial tiles) looped over a
 * whole index space by user code, template.instantiate or the CLI
 * (cli.py:166-198).  Each entry point below replaces such a loop with one
 * stream-ordered launch; INTEGRATION.md shows the ctypes binding the
 * reference would add.
 *
 * Conventions: every function returns lego_status (0 = OK) and never throws;
 * lego_last_error() holds a thread-local message for the last failure.  All
 * device buffers are owned by the caller (the Python side uses PyTorch only
 * for allocation and streams); `stream` is a cudaStream_t (NULL = legacy
 * default stream).  Calls are asynchronous with respect to the host.
 */
#ifndef LEGO_B200_H
#define LEGO_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LEGO_ABI_VERSION 1

/* Status codes map 1:1 onto the reference exception classes
 * (errors.py:4-83) where one exists. */
typedef enum {
    LEGO_OK = 0,
    LEGO_E_ARITY = 1,        /* ArityMismatch        */
    LEGO_E_BOUNDS = 2,       /* OutOfBounds          */
    LEGO_E_SHAPE = 3,        /* ShapeMismatch        */
    LEGO_E_UNSUPPORTED = 4,  /* UnsupportedNode      */
    LEGO_E_CUDA = 5,         /* CUDA runtime/driver  */
    LEGO_E_NVRTC = 6,        /* kernel JIT failed    */
    LEGO_E_BIJECTIVITY = 7,  /* BijectivityViolation */
    LEGO_E_ARG = 8           /* invalid argument     */
} lego_status;

/* A loaded program: one generated layout lowering (index maps and/or a
 * remap kernel) compiled for sm_100a. */
typedef struct lego_program_s *lego_program;

/* What a program holds; fixed at load time. */
typedef enum {
    LEGO_PROG_INDEX_MAP = 0,   /* lego_apply_map / lego_inv_map / lego_check_bijective */
    LEGO_PROG_GATHER = 1,      /* remap: dst[f] = src[g(f)], per-element g             */
    LEGO_PROG_TRANSPOSE = 2,   /* remap: digit-permutation, register-tiled transpose   */
    LEGO_PROG_BAND = 3,        /* remap: anti-diagonal band tiles through shared memory */
    LEGO_PROG_SCATTER = 4,     /* remap into an injective layout: dst[apply(x)] = src[x] */
    LEGO_PROG_STAGED = 5,      /* remap: per-block source box staged through smem      */
    LEGO_PROG_NW = 6,          /* Needleman-Wunsch wavefront over a LEGO tile layout   */
    LEGO_PROG_SOFTMAX = 7      /* row softmax with a LEGO thread/data layout           */
} lego_program_kind;

/* Program geometry.  Index-map programs: n = logical size, units = physical
 * size.  Remap programs: n = destination elements per matrix (source
 * elements for SCATTER), units = CTAs per matrix (grid.x; grid.y = batch).
 * NW programs: n = matrix side, units = tile rows H (= n for column strips),
 * reserved = 1 when tiles publish bottom rows (more than one tile row).
 * Softmax programs: n = row length (cols), units = rows the layout covers. */

typedef struct {
    int32_t kind;          /* lego_program_kind                                  */
    int32_t elem_bytes;    /* remap element size (1, 2, 4, 8, 16); 0 for maps   */
    int64_t n;             /* see above                                         */
    int64_t units;         /* see above                                         */
    int32_t unit_threads;  /* threads per work unit (1 or 32)                   */
    int32_t block;         /* threads per CTA                                   */
    int32_t smem_bytes;    /* dynamic shared memory per CTA                     */
    int32_t reserved;      /* remap alignment flags: LEGO_ALIGN_SRC_FREE (1) /  */
                           /* LEGO_ALIGN_DST_FREE (2) = that side's base and    */
                           /* batch stride need only element alignment; else   */
                           /* 16 bytes (vector access)                         */
} lego_program_info;

#define LEGO_ALIGN_SRC_FREE 1
#define LEGO_ALIGN_DST_FREE 2
/* scatter programs built with a fill mode (lego_remap_fill): FUSED = one
 * kernel writes every destination position (affine injective layouts,
 * whole 16-byte sectors); PASS = a vector fill, then the scatter */
#define LEGO_FILL_FUSED 4
#define LEGO_FILL_PASS 8

int32_t lego_abi_version(void);
const char *lego_last_error(void);

/* Device properties the host lowering needs (SM count, L2 bytes, CC). */
lego_status lego_device_info(int32_t device, int32_t *sm_count, int64_t *l2_bytes,
                             int32_t *cc_major, int32_t *cc_minor);

/* --- kernel JIT: CUDA C++ text -> sm_100a cubin (NVRTC) ------------------ */
/* Replaces reference emit.emit_expr(..., profile) (emit.py:90-102) as the
 * last step of the lowering: the text is a generated device function spliced
 * into a hand-written kernel template.  *cubin is freed with lego_free. */
lego_status lego_nvrtc_compile(const char *source, size_t source_len, const char *arch,
                               void **cubin, size_t *cubin_len, char *log, size_t log_cap);
void lego_free(void *p);

lego_status lego_program_load(const void *cubin, size_t cubin_len, const lego_program_info *info,
                              lego_program *out);
void lego_program_release(lego_program p);

/* --- user modules ---------------------------------------------------------
 * Kernels a user writes as LEGO templates (template.instantiate with
 * [target] cuda, reference template.py:444-537 + the new cuda profile of
 * emit.py), compiled by lego_nvrtc_compile, loaded into the current
 * device's primary context and launched by name; args as for
 * cuLaunchKernel (an array of pointers to the argument values). */
typedef struct lego_module_s *lego_module;
lego_status lego_module_load(const void *cubin, size_t cubin_len, lego_module *out);
void lego_module_release(lego_module m);
lego_status lego_module_launch(lego_module m, const char *kernel, uint32_t gx, uint32_t gy, uint32_t gz,
                               uint32_t bx, uint32_t by, uint32_t bz, uint32_t smem, void **args,
                               void *stream);

/* --- bulk layout evaluation ---------------------------------------------- */
/* out[k] = apply(canon_unflatten(dims, first + k))  for k < count
 *   (a loop of GroupBy.apply, layout.py:313; ExpandBy masks give -1)
 * out_bytes = 4 (int32) or 8 (int64). */
lego_status lego_apply_map(lego_program p, void *out, int32_t out_bytes, int64_t first,
                           int64_t count, void *stream);
/* out[k] = canon_flatten(dims, inv(first + k))  (a loop of GroupBy.inv, layout.py:320) */
lego_status lego_inv_map(lego_program p, void *out, int32_t out_bytes, int64_t first,
                         int64_t count, void *stream);
/* Proves the layout's apply is a bijection onto [0, n) by a device-side
 * histogram (validate() only checks GenPs up to 4096 points, layout.py:718).
 * hist: caller scratch of n uint32; *violations (host) = number of positions
 * hit != 1 times.  Synchronises the stream. */
lego_status lego_check_bijective(lego_program p, uint32_t *hist, int64_t *violations,
                                 void *stream);
/* The same histogram, counting positions hit more than once: the
 * injectivity proof of an injective-mode layout (layout.py:304-311), whose
 * unhit positions are legal.  Run before a scatter through a user GenP the
 * reference would only "trust". */
lego_status lego_check_injective(lego_program p, uint32_t *hist, int64_t *violations,
                                 void *stream);

/* --- layout remap (the data movement the index maps describe) ------------- */
/* For batch b < batch:  dst[b*dst_stride + f] = src[b*src_stride + g(f)]
 * with g = src.apply o dst.inv compiled into the program, i.e. for every
 * logical index x: dst[dst.apply(x)] = src[src.apply(x)].  Strides are in
 * elements; buffers and batch strides must be 16-byte aligned on the sides
 * the program accesses with vectors (see lego_program_info.reserved).
 * Routed programs (built with a destination routing, e.g. the fused
 * cross-rank transpose of shard.transpose_rows_fused): dst is a device array
 * of per-peer base addresses and destination element f is stored at
 * peer route.peer(f), element offset route.off(f); batch must be 1. */
lego_status lego_remap(lego_program p, const void *src, void *dst, int64_t batch,
                       int64_t src_stride, int64_t dst_stride, void *stream);
/* Scatter into an injective-mode layout writing EVERY destination position:
 * dst[apply(x)] = src[x], all other positions = *fill (elem_bytes bytes).
 * Replaces "zero the destination, then scatter" (whose partial-sector
 * stores force DRAM read-for-merge) for programs built with a fill mode. */
lego_status lego_remap_fill(lego_program p, const void *src, void *dst, int64_t batch,
                            int64_t src_stride, int64_t dst_stride, const void *fill, void *stream);

/* --- fixed kernels with LEGO-derived layouts ------------------------------ */
/* Row softmax, fp32, rows x cols row-major.  Rows in registers with float4
 * access when cols % 4 == 0 and both buffers are 16-byte aligned; any other
 * shape takes a scalar two-pass kernel (4-byte alignment). */
lego_status lego_softmax_f32(const float *x, float *y, int64_t rows, int64_t cols, void *stream);

/* The register-resident softmax through a program generated from the LEGO
 * thread/data layout GroupBy([R], [cols/(4T)], [T], [4]).OrderBy(Row(R, cols))
 * (kernels.softmax_program, LEGO_PROG_SOFTMAX; T = 256, cols % 4T == 0):
 * the kernel reads and writes element (row, it, tid, v) at the layout's
 * apply(row, it, tid, v).  cols must equal the program's, rows <= R,
 * buffers 16-byte aligned. */
lego_status lego_softmax_run(lego_program p, const float *x, float *y, int64_t rows, int64_t cols,
                             void *stream);
/* Test support: the float offsets the program's kernel accesses for the
 * first `rows` rows, out[(row*ITS + it)*T + tid] (int64, -1 past the row). */
lego_status lego_softmax_offsets(lego_program p, int64_t *out, int64_t rows, void *stream);

/* Needleman-Wunsch score matrix: score is (n+1) x (n+1) int32, row-major;
 * sim is n x n; batch independent alignments back to back.
 * S[0][j] = -j*p, S[i][0] = -i*p,
 * S[i][j] = max(S[i-1][j-1] + sim[i-1][j-1], S[i-1][j] - p, S[i][j-1] - p).
 * Column strips of 128 columns, each swept anti-diagonally by one CTA
 * (the default layout of lego_nw_run, built into the library).
 * The kernel works on offset scores S + (i+j)p in int32: requires
 * |p| * (2n + 2) < 2^30 (else LEGO_E_ARG) and scores within +-2^30.
 * sim must be 16-byte aligned.  Stream-ordered; keeps a per-(device, stream)
 * scratch buffer of strips x n int32 between calls. */
lego_status lego_nw_i32(const int32_t *sim, int32_t *score, int64_t n, int32_t penalty,
                        int64_t batch, void *stream);

/* Column band of the strip-mode recurrence: strips [strip_begin, strip_end)
 * (128 columns each) of every matrix, written into the full-size score; the
 * multi-GPU single-alignment path (one band per GPU, paper_2505_08091_b200
 * shard.nw_score_banded).  bnd_words: this band's right-edge columns, batch x
 * (strip_end - strip_begin) x n_pad int32 (n_pad = n rounded up to 32),
 * 16-byte aligned, preset by the caller to bytes 0x80 before any band that
 * reads it starts; left_words: the previous band's last edge column (matrix b
 * at left_words + b * left_batch_stride; a peer GPU's memory over NVLink), or
 * NULL when strip_begin == 0.  Edges are stored and polled at system scope.
 * max_ctas > 0 caps the persistent grid (bands sharing one GPU must all be
 * resident).  Other rules as lego_nw_i32.  Replaces no reference interface
 * (the reference has no NW kernel; SURVEY.md 8(e) "next" row). */
lego_status lego_nw_band_i32(const int32_t *sim, int32_t *score, int64_t n, int32_t penalty,
                             int64_t batch, int64_t strip_begin, int64_t strip_end, int32_t *bnd_words,
                             const int32_t *left_words, int64_t left_batch_stride, int32_t max_ctas,
                             void *stream);

/* The same recurrence through a program generated from a LEGO layout of the
 * cell grid (kernels.nw_layout / nw_program, LEGO_PROG_NW):
 *   GroupBy([NR*H, NC*128]).OrderBy(RegP([NR,H,NC,128],[1,3,2,4])).OrderBy(T, I)
 * T (over the NR x NC tile grid) is the order in which CTAs claim tiles, I
 * (over a tile's H x 128 cells) the shared-memory order of its rows.  The
 * host proves T a topological order of the tile dependencies and I
 * row-preserving with 16-byte lane groups before building the program.
 * n must equal the program's n; otherwise as lego_nw_i32. */
lego_status lego_nw_run(lego_program p, const int32_t *sim, int32_t *score, int64_t n,
                        int32_t penalty, int64_t batch, void *stream);

/* bf16 GEMM on tcgen05/TMEM: C[b] = A[b] * B[b]^T-free layouts:
 * A is M x K row-major, B is N x K row-major ("TN"), C is M x N row-major
 * bf16, fp32 accumulation.  raster: 0 = row-major CTA order, G > 0 = the
 * LEGO grouped raster GroupBy([MB/G, NB, G]).OrderBy(Row(MB/G, NB, G)) over
 * output tiles (G m-blocks of 128 rows per group).  Requires N % 8 == 0 and
 * K % 8 == 0 (16-byte rows); M, N, K need not be tile multiples (TMA
 * zero-fills the operand tails, the epilogue masks the stores).  The CTA-pair
 * kernel (cta_group::2, 256 x 512 or 256 x 256 tiles per 2-SM cluster) runs
 * for M % 256 == 0 and for ragged shapes; M % 256 == 128 with exact N, K
 * tiles takes the single-CTA 128 x 256 kernel (LEGO_GEMM_PAIR=0 forces it
 * for all exact shapes). */
lego_status lego_gemm_bf16(const void *A, const void *B, void *C, int64_t M, int64_t N,
                           int64_t K, int64_t batch, int32_t raster, void *stream);

/* Test support: the GEMM kernels' tile order, out[3t..3t+2] = (batch, m-block,
 * n-block) of tile t < mtiles*ntiles*batch, from the same device function
 * the kernels use (raster = G > 0: grouped raster of G m-blocks; 0:
 * row-major).  The single-CTA kernel passes m-blocks of 128 rows and G; the
 * CTA-pair kernel m-blocks of 256 rows and G / 2. */
lego_status lego_gemm_raster(int32_t *out, int64_t mtiles, int64_t ntiles, int64_t batch, int32_t raster,
                             void *stream);

/* The four data-layout variants of the paper's LEGO matmul (Row vs Col
 * layouts of each operand): a_major / b_major = 0 keeps
 * the operand K-major (A: M x K, B: N x K row-major, as above), 1 makes it
 * MN-major (A stored K x M, B stored K x N row-major), fed to tcgen05 as an
 * MN-major UMMA operand (no transpose pass).  MN-major A needs M % 8 == 0;
 * K % 8 == 0 is needed only while an operand is K-major. */
lego_status lego_gemm_bf16_ex(const void *A, const void *B, void *C, int64_t M, int64_t N,
                              int64_t K, int64_t batch, int32_t raster, int32_t a_major,
                              int32_t b_major, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* LEGO_B200_H */
