/*
 * oracle/orc.c -- CPU ORACLE (test infrastructure, NOT the product path).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * leg may load this library.  It shares no code, header, table or constant generator with
 * the CUDA product package and never includes or links anything from it.
 *
 * What it computes (each function cites the passage it follows):
 *   orc_sm64            SplitMix64 output k of a stream keyed by `key` (workload generator,
 *                       reading Q9 of DESIGN.md; pinned by the published SplitMix64 test vector).
 *   orc_rmat_edges      R-MAT edge list (BASELINE configs 1/4/5; reading Q9).
 *   orc_er_edges        Erdos-Renyi G(n,m) edge list (BASELINE config 3; reading Q11).
 *   orc_build_csr       AT in CSR (rows = destination, cols = source, ascending, unique, no
 *                       self-loops) and out_degree (Fig. 6 inputs `AT`,
 *                       `out_degree`; SPEC.md:57-58 CSR invariants; reading Q8/Q12).
 *   orc_pagerank_f32/64 The PageRank sweep of PAPER.md Fig. 6 (lines 272-294) in the paper's
 *                       order, with the dangling-mass readings Q1 (UNIFORM | DROP), Q2 (reciprocal
 *                       scaling), Q3 (constants in double, rounded once), Q4 (fp64 accumulation),
 *                       Q5/Q6 (loop test).  Plain loops, ascending index order.
 *   orc_mxv_plus_f32/64 plus-second mxv over a pattern CSR, fp64 row sums.
 *
 * Compile with -O2 -ffp-contract=off (no FMA contraction, no fast-math): every float
 * operation below is one IEEE-754 round-to-nearest operation in the written type.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

/* ---------------------------------------------------------------- generators */

/* SplitMix64 (Steele, Lea, Flood 2014): output k of the stream whose state starts at `key`:
 * z = key + (k+1)*gamma, then the standard finaliser. */
uint64_t orc_sm64(uint64_t key, uint64_t k)
{
    uint64_t z = key + (k + 1u) * 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/* R-MAT (a,b,c,d) = (0.57, 0.19, 0.19, 0.05), BASELINE configs 1/4/5.
 * Edge e, level l = 0..scale-1 (l = 0 decides the most significant bit):
 *   u = sm64(seed, e*64 + l) >> 11   (53 bits)
 *   u <  floor(0.57*2^53)           -> quadrant (0,0)
 *   u <  floor(0.76*2^53)           -> (0,1)
 *   u <  floor(0.95*2^53)           -> (1,0)
 *   else                            -> (1,1)
 * (row bit, col bit) = (src bit, dst bit).  No noise, no permutation. */
void orc_rmat_edges(int scale, int64_t m, uint64_t seed, int32_t *src, int32_t *dst)
{
    const uint64_t A = 5134103575202365ULL;     /* floor(0.57 * 2^53) */
    const uint64_t AB = 6845471433603153ULL;    /* floor(0.76 * 2^53) */
    const uint64_t ABC = 8556839292003942ULL;   /* floor(0.95 * 2^53) */
    for (int64_t e = 0; e < m; e++) {
        uint32_t s = 0, d = 0;
        for (int l = 0; l < scale; l++) {
            uint64_t u = orc_sm64(seed, (uint64_t)e * 64u + (uint64_t)l) >> 11;
            uint32_t sbit, dbit;
            if (u < A) { sbit = 0; dbit = 0; }
            else if (u < AB) { sbit = 0; dbit = 1; }
            else if (u < ABC) { sbit = 1; dbit = 0; }
            else { sbit = 1; dbit = 1; }
            s |= sbit << (scale - 1 - l);
            d |= dbit << (scale - 1 - l);
        }
        src[e] = (int32_t)s;
        dst[e] = (int32_t)d;
    }
}

/* Erdos-Renyi G(n, m), n = 2^logn: src = top logn bits of sm64(seed, 2e),
 * dst = top logn bits of sm64(seed, 2e+1) (BASELINE config 3, reading Q11). */
void orc_er_edges(int logn, int64_t m, uint64_t seed, int32_t *src, int32_t *dst)
{
    for (int64_t e = 0; e < m; e++) {
        src[e] = (int32_t)(orc_sm64(seed, 2u * (uint64_t)e) >> (64 - logn));
        dst[e] = (int32_t)(orc_sm64(seed, 2u * (uint64_t)e + 1u) >> (64 - logn));
    }
}

/* ---------------------------------------------------------------- CSR build */

/* Edge u->v is stored at AT[v,u] (PAPER.md:266 `AT`; reading Q8).  Canonical form (Q12):
 * rows ascending, columns strictly ascending within a row, duplicates removed, self-loops
 * dropped.  deg[u] = number of stored entries in column u of AT = out-degree of u.
 * Two stable counting sorts (by src, then by dst) order the edges by (dst, src);
 * the rest is one pass.  rowptr must hold n+1 entries; colidx must hold m entries
 * (the function returns nnz <= m).  Returns -1 on allocation failure. */
int64_t orc_build_csr(int64_t n, int64_t m, const int32_t *src, const int32_t *dst,
                      int64_t *rowptr, int32_t *colidx, int32_t *deg)
{
    int64_t *cnt = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
    int64_t *tmp = (int64_t *)malloc((size_t)(m > 0 ? m : 1) * sizeof(int64_t));
    int64_t *ord = (int64_t *)malloc((size_t)(m > 0 ? m : 1) * sizeof(int64_t));
    if (!cnt || !tmp || !ord) { free(cnt); free(tmp); free(ord); return -1; }

    /* pass 1: stable counting sort of edge ids by src */
    for (int64_t e = 0; e < m; e++) cnt[src[e] + 1]++;
    for (int64_t i = 0; i < n; i++) cnt[i + 1] += cnt[i];
    for (int64_t e = 0; e < m; e++) tmp[cnt[src[e]]++] = e;
    /* pass 2: stable counting sort of those ids by dst */
    memset(cnt, 0, ((size_t)n + 1) * sizeof(int64_t));
    for (int64_t e = 0; e < m; e++) cnt[dst[e] + 1]++;
    for (int64_t i = 0; i < n; i++) cnt[i + 1] += cnt[i];
    for (int64_t q = 0; q < m; q++) { int64_t e = tmp[q]; ord[cnt[dst[e]]++] = e; }

    /* one pass: drop self-loops and adjacent duplicates, count rows and degrees */
    for (int64_t i = 0; i < n; i++) deg[i] = 0;
    for (int64_t i = 0; i <= n; i++) rowptr[i] = 0;
    int64_t nnz = 0;
    int64_t prev_d = -1, prev_s = -1;
    for (int64_t q = 0; q < m; q++) {
        int64_t e = ord[q];
        int64_t d = dst[e], s = src[e];
        if (s == d) continue;                       /* self-loop */
        if (d == prev_d && s == prev_s) continue;   /* duplicate */
        prev_d = d; prev_s = s;
        colidx[nnz++] = (int32_t)s;
        rowptr[d + 1]++;
        deg[s]++;
    }
    for (int64_t i = 0; i < n; i++) rowptr[i + 1] += rowptr[i];
    free(cnt); free(tmp); free(ord);
    return nnz;
}

/* ---------------------------------------------------------------- mxv */

/* m[i] = (T) sum_{p in row i, ascending} (double) x[colidx[p]]  (plus-second semiring on the
 * pattern matrix; empty row -> identity 0). */
void orc_mxv_plus_f64(int64_t n, const int64_t *rowptr, const int32_t *colidx,
                      const double *x, double *m)
{
    for (int64_t i = 0; i < n; i++) {
        double acc = 0.0;
        for (int64_t p = rowptr[i]; p < rowptr[i + 1]; p++) acc += x[colidx[p]];
        m[i] = acc;
    }
}

void orc_mxv_plus_f32(int64_t n, const int64_t *rowptr, const int32_t *colidx,
                      const float *x, float *m)
{
    for (int64_t i = 0; i < n; i++) {
        double acc = 0.0;
        for (int64_t p = rowptr[i]; p < rowptr[i + 1]; p++) acc += (double)x[colidx[p]];
        m[i] = (float)acc;
    }
}

/* ---------------------------------------------------------------- PageRank */

/* PAPER.md Fig. 6 (lines 266-294), step by step:
 *   r   = GrBVector(n, 1/n)                              line 277   (constant rounded once to T)
 *   d   = max(deg/alpha, 1/alpha);  r = t / d             lines 278-286
 *         -> reading Q2: y = t * dinv,  dinv = (T)(alpha/deg) or 0 when deg == 0
 *   r   = mxv(0, +, second, AT, y)                        line 287   (fp64 row sums, Q4)
 *   r   = ewise_add(+, rt, r)                             line 288   rt = (1-alpha)/n
 *         + dangling mass alpha*ds/n when variant == UNIFORM (Q1, BASELINE config 4);
 *         the constant c = (T)((alpha/n)*ds + (1-alpha)/n) is formed in double, rounded once (Q3)
 *   t   = ewise_add(|x-y|, t, r); rdiff = reduce(+, t)    lines 290-291  (fp64 sum, Q4)
 *   loop while iter <= itermax && rdiff > tol             line 284   (Q5/Q6: tol < 0 => fixed count)
 * ds (UNIFORM) = sum over dangling j (deg[j] == 0) of the previous ranks, ascending j.
 * Outputs: r (T[n]), delta_hist[k-1] = rdiff after sweep k, ds_hist[k-1] = ds used by sweep k.
 * Returns the number of sweeps (SpMVs); Fig. 6's `iter` is sweeps + 1. */
#define ORC_PAGERANK(NAME, T)                                                              \
int NAME(int64_t n, const int64_t *rowptr, const int32_t *colidx, const int32_t *deg,     \
         double alpha, int uniform, int itermax, double tol,                               \
         T *r_out, double *delta_hist, double *ds_hist)                                    \
{                                                                                          \
    T *dinv = (T *)malloc((size_t)n * sizeof(T));                                          \
    T *r = (T *)malloc((size_t)n * sizeof(T));                                             \
    T *t = (T *)malloc((size_t)n * sizeof(T));                                             \
    T *y = (T *)malloc((size_t)n * sizeof(T));                                             \
    if (!dinv || !r || !t || !y) { free(dinv); free(r); free(t); free(y); return -1; }     \
    for (int64_t j = 0; j < n; j++)                                                        \
        dinv[j] = deg[j] > 0 ? (T)(alpha / (double)deg[j]) : (T)0;                         \
    const T r0 = (T)(1.0 / (double)n);                                                     \
    for (int64_t i = 0; i < n; i++) r[i] = r0;                                             \
    const double tele = (1.0 - alpha) / (double)n;                                         \
    const double a_n = alpha / (double)n;                                                  \
    int sweeps = 0;                                                                        \
    for (int k = 1; k <= itermax; k++) {                                                   \
        double ds = 0.0;                                                                   \
        for (int64_t j = 0; j < n; j++) if (deg[j] == 0) ds += (double)r[j];               \
        for (int64_t i = 0; i < n; i++) t[i] = r[i];                                       \
        for (int64_t j = 0; j < n; j++) y[j] = t[j] * dinv[j];                             \
        const T c = uniform ? (T)(a_n * ds + tele) : (T)tele;                              \
        /* rows are independent: the OpenMP build (liborc_omp.so, cpu_baseline only)     \
         * splits them over threads; every row's sum keeps its ascending order, so the     \
         * result is identical to the single-threaded build */                             \
        _Pragma("omp parallel for schedule(static)")                                       \
        for (int64_t i = 0; i < n; i++) {                                                  \
            double acc = 0.0;                                                              \
            for (int64_t p = rowptr[i]; p < rowptr[i + 1]; p++) acc += (double)y[colidx[p]]; \
            const T mi = (T)acc;                                                           \
            r[i] = mi + c;                                                                 \
        }                                                                                  \
        double delta = 0.0;                                                                \
        for (int64_t i = 0; i < n; i++) {                                                  \
            T e = r[i] - t[i];                                                             \
            if (e < 0) e = -e;                                                             \
            delta += (double)e;                                                            \
        }                                                                                  \
        if (delta_hist) delta_hist[k - 1] = delta;                                         \
        if (ds_hist) ds_hist[k - 1] = ds;                                                  \
        sweeps = k;                                                                        \
        if (tol >= 0.0 && !(delta > tol)) break;                                           \
    }                                                                                      \
    memcpy(r_out, r, (size_t)n * sizeof(T));                                               \
    free(dinv); free(r); free(t); free(y);                                                 \
    return sweeps;                                                                         \
}

ORC_PAGERANK(orc_pagerank_f64, double)
ORC_PAGERANK(orc_pagerank_f32, float)

/* One sweep over a row block [lo, hi) only (used by the CPU model of the 1-D row partition,
 * DESIGN.md "multi-GPU"): r[i - lo] = (T)(rowsum_i) + c for i in [lo, hi). */
void orc_sweep_rows_f32(int64_t lo, int64_t hi, const int64_t *rowptr, const int32_t *colidx,
                        const float *y, float c, float *r_block)
{
    for (int64_t i = lo; i < hi; i++) {
        double acc = 0.0;
        for (int64_t p = rowptr[i]; p < rowptr[i + 1]; p++) acc += (double)y[colidx[p]];
        const float mi = (float)acc;
        r_block[i - lo] = mi + c;
    }
}
