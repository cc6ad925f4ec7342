/*
 * lego_oracle.c -- CPU restatement of the reference LEGO layout algebra.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the B200
 * backend: only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg may load it.  The product path never links or calls
 * it (and fails loudly when its own CUDA library is missing).
 *
 * Every function restates one reference function, cited file:line against
 * /root/reference/pkg/src/lego/.  Arithmetic is int64 with floor semantics
 * (the reference uses Python ints, floor // and %): every operand of / and %
 * on these paths is a non-negative index, where C truncation equals floor.
 *
 * Parity is pinned by tests/test_oracle.py against golden vectors produced
 * by the reference itself (tests/golden/make_golden.py).
 *
 * Layout descriptor (int64 array, produced by oracle/oracle.py):
 *   [0] 0x4C45474F ("LEGO")  [1] 1 (version)
 *   [2] kind: 0 = GroupBy, 1 = ExpandBy
 *   ExpandBy: rank, physical[rank], expanded[rank], then a GroupBy body
 *   GroupBy body: d, dims[d], nstages, then per stage: nperms, per perm:
 *       pkind (0 RegP, 1 identity, 2 rev, 3 antidiag), rank, shape[rank],
 *       and for RegP sigma[rank] (1-based)
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define MAXR 16
#define MAXP 16
#define MAXS 16

enum { P_REGP = 0, P_IDENTITY = 1, P_REV = 2, P_ANTIDIAG = 3 };

typedef struct {
    int kind, rank;
    int64_t shape[MAXR];
    int64_t sigma[MAXR];          /* 1-based, RegP only */
} perm_t;

typedef struct {
    int nperms;
    perm_t perms[MAXP];
    int rank;                     /* concatenated dims */
    int64_t dims[MAXR];
} stage_t;

typedef struct {
    int d;
    int64_t dims[MAXR];
    int nstages;
    stage_t stages[MAXS];
    /* ExpandBy wrapper */
    int expand, erank;
    int64_t physical[MAXR], expanded[MAXR];
    int64_t size;                 /* GroupBy: logical size; ExpandBy: physical size */
} layout_t;

/* ---- canonical bijections: layout.py:93-106 (flatten), :109-123 (unflatten) */

static int64_t canon_flatten(int rank, const int64_t *shape, const int64_t *idx) {
    int64_t acc = 0;
    for (int k = 0; k < rank; ++k) acc = acc * shape[k] + idx[k];   /* Horner == sum c*stride */
    return acc;
}

static void canon_unflatten(int rank, const int64_t *shape, int64_t flat, int64_t *out) {
    /* innermost first with % and //, leading coordinate is the bare quotient */
    for (int k = rank - 1; k >= 1; --k) { out[k] = flat % shape[k]; flat /= shape[k]; }
    out[0] = flat;
}

/* ---- RegP: layout.py:142-149 (apply flattens sigma-gathered idx in the
 *      sigma-gathered shape; inv unflattens and scatters back) */

static int64_t regp_apply(const perm_t *p, const int64_t *idx) {
    int64_t sh[MAXR], ix[MAXR];
    for (int k = 0; k < p->rank; ++k) { sh[k] = p->shape[p->sigma[k] - 1]; ix[k] = idx[p->sigma[k] - 1]; }
    return canon_flatten(p->rank, sh, ix);
}

static void regp_inv(const perm_t *p, int64_t flat, int64_t *out) {
    int64_t sh[MAXR], c[MAXR];
    for (int k = 0; k < p->rank; ++k) sh[k] = p->shape[p->sigma[k] - 1];
    canon_unflatten(p->rank, sh, flat, c);
    for (int k = 0; k < p->rank; ++k) out[p->sigma[k] - 1] = c[k];   /* gather by sigma^-1 */
}

/* ---- built-in GenPs: identity layout.py:524-533, reverse layout.py:536-548,
 *      antidiag layout.py:551-601 (Fig. 7 of the paper, transcribed) */

static int64_t isqrt64(int64_t x) {
    int64_t r = (int64_t)sqrt((double)x);
    while (r * r > x) --r;
    while ((r + 1) * (r + 1) <= x) ++r;
    return r;
}

static int64_t antidiag_fwd(int64_t n, int64_t i, int64_t j) {
    int64_t t = i + j + 1;                               /* layout.py:565 */
    if (t <= n) return i + t * (t - 1) / 2;              /* layout.py:566-567 */
    t = 2 * n - t;                                       /* layout.py:568 */
    return n * n - n + i - t * (t - 1) / 2;              /* layout.py:569 */
}

static void antidiag_inv(int64_t n, int64_t flat, int64_t *out) {
    int64_t half = n * (n + 1) / 2;
    int64_t x = flat < half ? flat : n * n - 1 - flat;   /* layout.py:581 */
    int64_t t = isqrt64(2 * x);                          /* layout.py:582 */
    if (x >= t * (t + 1) / 2) t += 1;                    /* layout.py:583-584 */
    int64_t i = x - t * (t - 1) / 2;                     /* layout.py:585 */
    int64_t j = t - i - 1;                               /* layout.py:586 */
    if (flat < half) { out[0] = i; out[1] = j; }
    else { out[0] = n - 1 - i; out[1] = n - 1 - j; }     /* layout.py:587-589 */
}

static int64_t perm_apply(const perm_t *p, const int64_t *idx) {
    int64_t m[MAXR];
    switch (p->kind) {
    case P_REGP: return regp_apply(p, idx);
    case P_IDENTITY: return canon_flatten(p->rank, p->shape, idx);
    case P_REV:
        for (int k = 0; k < p->rank; ++k) m[k] = p->shape[k] - 1 - idx[k];
        return canon_flatten(p->rank, p->shape, m);
    default: return antidiag_fwd(p->shape[0], idx[0], idx[1]);
    }
}

static void perm_inv(const perm_t *p, int64_t flat, int64_t *out) {
    switch (p->kind) {
    case P_REGP: regp_inv(p, flat, out); return;
    case P_IDENTITY: canon_unflatten(p->rank, p->shape, flat, out); return;
    case P_REV:
        canon_unflatten(p->rank, p->shape, flat, out);
        for (int k = 0; k < p->rank; ++k) out[k] = p->shape[k] - 1 - out[k];
        return;
    default: antidiag_inv(p->shape[0], flat, out); return;
    }
}

static int64_t perm_size(const perm_t *p) {
    int64_t s = 1;
    for (int k = 0; k < p->rank; ++k) s *= p->shape[k];
    return s;
}

/* ---- OrderBy: layout.py:237-247 (apply: acc*prod(dims)+cur outermost first),
 *      layout.py:249-258 (inv: peel innermost first) */

static int64_t stage_apply(const stage_t *s, const int64_t *idx) {
    int64_t acc = 0;
    int pos = 0;
    for (int q = 0; q < s->nperms; ++q) {
        const perm_t *p = &s->perms[q];
        acc = acc * perm_size(p) + perm_apply(p, idx + pos);
        pos += p->rank;
    }
    return acc;
}

static void stage_inv(const stage_t *s, int64_t flat, int64_t *out) {
    int pos = s->rank;
    for (int q = s->nperms - 1; q >= 0; --q) {
        const perm_t *p = &s->perms[q];
        int64_t sz = perm_size(p);
        pos -= p->rank;
        perm_inv(p, flat % sz, out + pos);
        flat /= sz;
    }
}

/* ---- GroupBy: layout.py:313-318 (apply: flatten, then stages in listed order),
 *      layout.py:320-328 (inv: stages in reverse, unflatten at the end) */

static int64_t group_apply_flat(const layout_t *L, int64_t x) {
    /* x is canon_flatten(dims, idx) of the logical index */
    int64_t c[MAXR];
    int64_t flat = x;
    for (int k = 0; k < L->nstages; ++k) {
        const stage_t *s = &L->stages[k];
        canon_unflatten(s->rank, s->dims, flat, c);
        flat = stage_apply(s, c);
    }
    return flat;
}

static int64_t group_inv_flat(const layout_t *L, int64_t f) {
    int64_t c[MAXR];
    for (int k = L->nstages - 1; k >= 0; --k) {
        const stage_t *s = &L->stages[k];
        stage_inv(s, f, c);
        f = canon_flatten(s->rank, s->dims, c);
    }
    return f;   /* == canon_flatten(dims, inv(f)) */
}

/* ---- ExpandBy: layout.py:383-393 (apply, -1 when masked), :395-400 (inv) */

static int64_t layout_apply_flat(const layout_t *L, int64_t x) {
    int64_t g = group_apply_flat(L, x);
    if (!L->expand) return g;
    int64_t c[MAXR];
    canon_unflatten(L->erank, L->expanded, g, c);
    for (int k = 0; k < L->erank; ++k)
        if (c[k] >= L->physical[k]) return -1;
    return canon_flatten(L->erank, L->physical, c);
}

static int64_t layout_inv_flat(const layout_t *L, int64_t f) {
    if (L->expand) {
        int64_t c[MAXR];
        canon_unflatten(L->erank, L->physical, f, c);
        f = canon_flatten(L->erank, L->expanded, c);
    }
    return group_inv_flat(L, f);
}

/* ---- descriptor decoding ------------------------------------------------ */

static int read_group(const int64_t *d, int64_t n, int64_t *at, layout_t *L) {
#define NEED(k) do { if (*at + (k) > n) return -1; } while (0)
    NEED(1);
    L->d = (int)d[(*at)++];
    if (L->d < 1 || L->d > MAXR) return -2;
    NEED(L->d);
    L->size = 1;
    for (int k = 0; k < L->d; ++k) { L->dims[k] = d[(*at)++]; L->size *= L->dims[k]; }
    NEED(1);
    L->nstages = (int)d[(*at)++];
    if (L->nstages < 0 || L->nstages > MAXS) return -3;
    for (int s = 0; s < L->nstages; ++s) {
        stage_t *st = &L->stages[s];
        NEED(1);
        st->nperms = (int)d[(*at)++];
        if (st->nperms < 1 || st->nperms > MAXP) return -4;
        st->rank = 0;
        for (int q = 0; q < st->nperms; ++q) {
            perm_t *p = &st->perms[q];
            NEED(2);
            p->kind = (int)d[(*at)++];
            p->rank = (int)d[(*at)++];
            if (p->rank < 1 || st->rank + p->rank > MAXR) return -5;
            NEED(p->rank);
            for (int k = 0; k < p->rank; ++k) { p->shape[k] = d[(*at)++]; st->dims[st->rank + k] = p->shape[k]; }
            if (p->kind == P_REGP) {
                NEED(p->rank);
                for (int k = 0; k < p->rank; ++k) p->sigma[k] = d[(*at)++];
            } else if (p->kind == P_ANTIDIAG) {
                if (p->rank != 2 || p->shape[0] != p->shape[1]) return -6;
            } else if (p->kind != P_IDENTITY && p->kind != P_REV) {
                return -7;
            }
            st->rank += p->rank;
        }
    }
    return 0;
#undef NEED
}

static int decode(const int64_t *d, int64_t n, layout_t *L) {
    memset(L, 0, sizeof(*L));
    if (n < 3 || d[0] != 0x4C45474F || d[1] != 1) return -10;
    int64_t at = 3;
    if (d[2] == 1) {
        L->expand = 1;
        if (at >= n) return -11;
        L->erank = (int)d[at++];
        if (L->erank < 1 || L->erank > MAXR || at + 2 * L->erank > n) return -12;
        for (int k = 0; k < L->erank; ++k) L->physical[k] = d[at++];
        for (int k = 0; k < L->erank; ++k) L->expanded[k] = d[at++];
    } else if (d[2] != 0) {
        return -13;
    }
    int rc = read_group(d, n, &at, L);
    if (rc) return rc;
    if (L->expand) {
        L->size = 1;
        for (int k = 0; k < L->erank; ++k) L->size *= L->physical[k];
    }
    return 0;
}

/* ---- exported bulk API ---------------------------------------------------- */

int oracle_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* thread count for the parallel loops (launchers such as torchrun preset
   OMP_NUM_THREADS=1; the timed CPU baseline wants every host core) */
void oracle_set_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

/* out[k] = apply(canon_unflatten(dims, first + k)); -1 marks an ExpandBy mask */
int oracle_apply_range(const int64_t *desc, int64_t ndesc, int64_t first, int64_t count, int64_t *out) {
    layout_t L;
    int rc = decode(desc, ndesc, &L);
    if (rc) return rc;
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < count; ++k) out[k] = layout_apply_flat(&L, first + k);
    return 0;
}

/* out[k] = canon_flatten(dims, inv(first + k)) */
int oracle_inv_range(const int64_t *desc, int64_t ndesc, int64_t first, int64_t count, int64_t *out) {
    layout_t L;
    int rc = decode(desc, ndesc, &L);
    if (rc) return rc;
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < count; ++k) out[k] = layout_inv_flat(&L, first + k);
    return 0;
}

/* Remap through two layouts over the same logical space, element by element:
 * for every logical index x, dst[dst.apply(x)] = src[src.apply(x)]
 * (ndesc == 0 for either side means the canonical row-major layout). */
int oracle_remap(const int64_t *src_desc, int64_t nsrc, const int64_t *dst_desc, int64_t ndst,
                 int64_t logical_size, const void *src, void *dst, int elem_bytes,
                 int64_t first, int64_t count) {
    layout_t S, D;
    int have_s = nsrc > 0, have_d = ndst > 0, rc;
    if (have_s && (rc = decode(src_desc, nsrc, &S))) return rc;
    if (have_d && (rc = decode(dst_desc, ndst, &D))) return rc;
    (void)logical_size;
    const char *s = (const char *)src;
    char *o = (char *)dst;
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < count; ++k) {
        int64_t x = first + k;
        int64_t ps = have_s ? layout_apply_flat(&S, x) : x;
        int64_t pd = have_d ? layout_apply_flat(&D, x) : x;
        if (ps >= 0 && pd >= 0) memcpy(o + pd * elem_bytes, s + ps * elem_bytes, (size_t)elem_bytes);
    }
    return 0;
}

/* ---- Needleman-Wunsch score matrix (restatement; the reference ships no
 *      NW code -- PAPER.md:1298-1301 cites Rodinia).  score is (n+1)^2:
 *      S[0][j] = -j*p, S[i][0] = -i*p,
 *      S[i][j] = max(S[i-1][j-1] + sim[i-1][j-1], S[i-1][j] - p, S[i][j-1] - p).
 *      Anti-diagonal sweep so OpenMP can split each diagonal. */
int oracle_nw(const int32_t *sim, int64_t n, int32_t p, int32_t *score) {
    const int64_t w = n + 1;
    for (int64_t j = 0; j <= n; ++j) score[j] = (int32_t)(-j * p);
    for (int64_t i = 0; i <= n; ++i) score[i * w] = (int32_t)(-i * p);
    for (int64_t t = 2; t <= 2 * n; ++t) {             /* i + j == t, 1 <= i, j <= n */
        int64_t lo = t - n > 1 ? t - n : 1, hi = t - 1 < n ? t - 1 : n;
#pragma omp parallel for schedule(static) if (hi - lo > 4096)
        for (int64_t i = lo; i <= hi; ++i) {
            int64_t j = t - i;
            int32_t d = score[(i - 1) * w + j - 1] + sim[(i - 1) * n + j - 1];
            int32_t u = score[(i - 1) * w + j] - p;
            int32_t l = score[i * w + j - 1] - p;
            int32_t m = d > u ? d : u;
            score[i * w + j] = m > l ? m : l;
        }
    }
    return 0;
}

/* Row-major NW, single thread, for small sizes (cross-checks the sweep). */
int oracle_nw_rowmajor(const int32_t *sim, int64_t n, int32_t p, int32_t *score) {
    const int64_t w = n + 1;
    for (int64_t j = 0; j <= n; ++j) score[j] = (int32_t)(-j * p);
    for (int64_t i = 1; i <= n; ++i) {
        score[i * w] = (int32_t)(-i * p);
        for (int64_t j = 1; j <= n; ++j) {
            int32_t d = score[(i - 1) * w + j - 1] + sim[(i - 1) * n + j - 1];
            int32_t u = score[(i - 1) * w + j] - p;
            int32_t l = score[i * w + j - 1] - p;
            int32_t m = d > u ? d : u;
            score[i * w + j] = m > l ? m : l;
        }
    }
    return 0;
}
