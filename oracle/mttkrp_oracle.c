/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct CPU reference for symmetric sparse MTTKRP.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * `--impl reference` leg may load this library.  The product path
 * (paper_2406_09266_b200/) never includes, links or calls it, and this file
 * includes nothing from the product path.
 *
 * What it computes ("plain definition"):
 *   The stored entries define a dense fully-symmetric tensor
 *     Abar[x] = sum over stored e with sort(x) == sort(idx_e) of v_e
 *   (Def. Symmetry; Def. Canonical),
 *   and the result is the naive, non-symmetric MTTKRP on it
 *     C[i,r] = sum_{j_1..j_{n-1}} Abar[i,j_1..j_{n-1}] * prod_t B[j_t, r]
 *   (MTTKRP definitions).
 *
 * Algorithm (north_star "expands every canonical entry to all n! permutations
 * (deduplicated) and runs the naive non-symmetric MTTKRP in fp64"):
 *   1. vals and B are widened fp32 -> fp64 (exact);
 *   2. for every stored entry e (any order, duplicates allowed):
 *        p = sort(idx_e)   (ascending),  v = vals_e;
 *   3. visit every DISTINCT permutation p of that multiset exactly once
 *      (the classic lexicographic next-permutation walk, which yields
 *      n!/prod m_r! permutations — PAPER.md:289-291 "we perform the same
 *      number of assignments as unique permutations of the indices");
 *   4. for each p and each r:  term = v * prod_{t=1}^{n-1} B[p_t, r];
 *        C[p_0, r] += term;   S[p_0, r] += |term|
 *      (one update per expanded non-zero: the naive kernel).
 *   S is the sum of absolute terms that normalises the parity error
 *   (BASELINE.json north_star).
 *
 * Threads: entries are split into contiguous slices; each thread owns a
 * private (C, S) copy that is summed at the end, or — when private copies
 * would exceed the memory budget — each thread scans every entry and keeps
 * only the permutations whose p_0 falls in its own row range.  Either way
 * the arithmetic per update is exactly step 4.
 *
 * Errors: returns 0 on success, 1 on bad arguments (order outside 1..8,
 * dim < 1, nnz < 0, R < 1, null pointers), 3 on an index outside [0, dim),
 * 5 when memory cannot be allocated.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORACLE_MAX_ORDER 8

/* Step 3: rearrange p[0..n) into the next lexicographically greater
 * permutation of its multiset; returns 0 when p was the last one. */
static int next_perm(int32_t *p, int n) {
    int i = n - 2;
    while (i >= 0 && p[i] >= p[i + 1]) i--;
    if (i < 0) return 0;
    int j = n - 1;
    while (p[j] <= p[i]) j--;
    int32_t t = p[i]; p[i] = p[j]; p[j] = t;
    for (int a = i + 1, b = n - 1; a < b; a++, b--) { t = p[a]; p[a] = p[b]; p[b] = t; }
    return 1;
}

static void sort_small(int32_t *p, int n) {
    for (int a = 1; a < n; a++) {
        int32_t x = p[a];
        int b = a - 1;
        while (b >= 0 && p[b] > x) { p[b + 1] = p[b]; b--; }
        p[b + 1] = x;
    }
}

typedef struct {
    int order; int64_t dim; int R;
    const int32_t *idx; const float *vals; const float *B;
    int64_t e_begin, e_end;      /* entry slice                                     */
    int64_t row_lo, row_hi;      /* only p_0 in [row_lo,row_hi) is kept             */
    const int32_t *rowslot;      /* optional: row -> output slot (-1 = drop)        */
    double *C, *S;               /* output rows indexed by (p_0 - row_lo) or slot   */
    double *term;                /* scratch [R]                                     */
} job_t;

static void *run_job(void *arg) {
    job_t *J = (job_t *)arg;
    const int n = J->order, R = J->R;
    int32_t p[ORACLE_MAX_ORDER];
    for (int64_t e = J->e_begin; e < J->e_end; e++) {
        for (int t = 0; t < n; t++) p[t] = J->idx[e * n + t];
        sort_small(p, n);                                   /* step 2 */
        const double v = (double)J->vals[e];                /* step 1 */
        do {                                                /* step 3 */
            int64_t row = p[0];
            int64_t out;
            if (J->rowslot) {
                out = J->rowslot[row];
                if (out < 0) continue;
            } else {
                if (row < J->row_lo || row >= J->row_hi) continue;
                out = row - J->row_lo;
            }
            for (int r = 0; r < R; r++) J->term[r] = v;     /* step 4 */
            for (int t = 1; t < n; t++) {
                const float *b = J->B + (int64_t)p[t] * R;
                for (int r = 0; r < R; r++) J->term[r] *= (double)b[r];
            }
            double *c = J->C + out * R, *s = J->S + out * R;
            for (int r = 0; r < R; r++) { c[r] += J->term[r]; s[r] += fabs(J->term[r]); }
        } while (next_perm(p, n));
    }
    return NULL;
}

static int check_args(int order, int64_t dim, int64_t nnz, const int32_t *idx,
                      const float *vals, const float *B, int R) {
    if (order < 1 || order > ORACLE_MAX_ORDER || dim < 1 || nnz < 0 || R < 1) return 1;
    if (nnz > 0 && (!idx || !vals)) return 1;
    if (!B) return 1;
    for (int64_t k = 0; k < nnz * order; k++)
        if (idx[k] < 0 || idx[k] >= dim) return 3;
    return 0;
}

/* Runs jobs[0..T) on T threads (job 0 on the calling thread). */
static void run_all(job_t *jobs, int T) {
    pthread_t *th = (pthread_t *)calloc((size_t)T, sizeof(pthread_t));
    int *started = (int *)calloc((size_t)T, sizeof(int));
    for (int k = 1; k < T; k++)
        started[k] = (pthread_create(&th[k], NULL, run_job, &jobs[k]) == 0);
    run_job(&jobs[0]);
    for (int k = 1; k < T; k++) {
        if (started[k]) pthread_join(th[k], NULL);
        else run_job(&jobs[k]);
    }
    free(th); free(started);
}

/*
 * Full oracle: C and S are [dim][R] fp64, overwritten.
 * nthreads <= 0 means 1.  mem_budget_bytes bounds the private copies
 * (0 = 8 GiB).
 */
int oracle_mttkrp(int order, int64_t dim, int64_t nnz, const int32_t *idx,
                  const float *vals, const float *B, int R, double *C, double *S,
                  int nthreads, int64_t mem_budget_bytes) {
    int rc = check_args(order, dim, nnz, idx, vals, B, R);
    if (rc) return rc;
    if (!C || !S) return 1;
    int T = nthreads > 0 ? nthreads : 1;
    if (mem_budget_bytes <= 0) mem_budget_bytes = (int64_t)8 << 30;
    const int64_t plane = dim * (int64_t)R;
    memset(C, 0, (size_t)plane * sizeof(double));
    memset(S, 0, (size_t)plane * sizeof(double));
    job_t *jobs = (job_t *)calloc((size_t)T, sizeof(job_t));
    double *scratch = (double *)calloc((size_t)T * R, sizeof(double));
    if (!jobs || !scratch) { free(jobs); free(scratch); return 5; }
    const int private_copies = T > 1 && (int64_t)T * plane * 16 <= mem_budget_bytes;
    double *priv = NULL;
    if (private_copies) {
        priv = (double *)calloc((size_t)(T - 1) * plane * 2, sizeof(double));
        if (!priv) { free(jobs); free(scratch); return 5; }
    }
    for (int k = 0; k < T; k++) {
        job_t *J = &jobs[k];
        J->order = order; J->dim = dim; J->R = R; J->idx = idx; J->vals = vals; J->B = B;
        J->term = scratch + (int64_t)k * R;
        J->rowslot = NULL;
        if (T == 1) {
            J->e_begin = 0; J->e_end = nnz; J->row_lo = 0; J->row_hi = dim; J->C = C; J->S = S;
        } else if (private_copies) {          /* entry slices, private outputs */
            J->e_begin = nnz * k / T; J->e_end = nnz * (k + 1) / T;
            J->row_lo = 0; J->row_hi = dim;
            if (k == 0) { J->C = C; J->S = S; }
            else { J->C = priv + (int64_t)(k - 1) * plane * 2; J->S = J->C + plane; }
        } else {                               /* row ownership, shared output */
            J->e_begin = 0; J->e_end = nnz;
            J->row_lo = dim * k / T; J->row_hi = dim * (k + 1) / T;
            J->C = C + J->row_lo * R; J->S = S + J->row_lo * R;
        }
    }
    run_all(jobs, T);
    if (private_copies) {
        for (int k = 1; k < T; k++) {
            const double *pc = priv + (int64_t)(k - 1) * plane * 2, *ps = pc + plane;
            for (int64_t q = 0; q < plane; q++) { C[q] += pc[q]; S[q] += ps[q]; }
        }
    }
    free(priv); free(jobs); free(scratch);
    return 0;
}

/*
 * The symmetric METHOD on the CPU, single thread, fp64 — not the oracle's
 * definition but the paper's algorithm written out plainly, for pin P4 (vs
 * the expansion above) and for the one-core CPU analogue of the paper's own
 * experiment (symmetric vs naive on one core; SURVEY.md
 * §8(d)).  For every stored entry: p = sort(idx_e), v = vals_e; the runs of
 * equal values have multiplicities m_w; for every run-first position u,
 *   coef_u = (n-1)! * m_u / prod_w m_w!            (distinct permutations of
 *            the multiset that put p_u first)
 *   C[p_u, r] += coef_u * v * prod_{s != u} B[p_s, r]
 * (fig:mttkrp_symmetrization_3 / Listing 6, after
 * distributive grouping).  C is [dim][R], overwritten.
 */
int oracle_mttkrp_symmetric(int order, int64_t dim, int64_t nnz, const int32_t *idx, const float *vals,
                            const float *B, int R, double *C) {
    int rc = check_args(order, dim, nnz, idx, vals, B, R);
    if (rc) return rc;
    if (!C) return 1;
    memset(C, 0, (size_t)(dim * (int64_t)R) * sizeof(double));
    double fact[ORACLE_MAX_ORDER + 1];
    fact[0] = 1.0;
    for (int k = 1; k <= ORACLE_MAX_ORDER; k++) fact[k] = fact[k - 1] * k;
    for (int64_t e = 0; e < nnz; e++) {
        int32_t p[ORACLE_MAX_ORDER];
        for (int t = 0; t < order; t++) {
            p[t] = idx[e * order + t];
            if (p[t] < 0 || p[t] >= dim) return 3;
        }
        sort_small(p, order);
        int mult[ORACLE_MAX_ORDER];            /* run length of the run starting at t (0 elsewhere) */
        double denom = 1.0;
        for (int t = 0; t < order;) {
            int u = t;
            while (u < order && p[u] == p[t]) u++;
            for (int q = t; q < u; q++) mult[q] = 0;
            mult[t] = u - t;
            denom *= fact[u - t];
            t = u;
        }
        const double v = (double)vals[e];
        for (int u = 0; u < order; u++) {
            if (mult[u] == 0) continue;
            const double coef = fact[order - 1] * mult[u] / denom;
            for (int r = 0; r < R; r++) {
                double prod = coef * v;
                for (int s = 0; s < order; s++)
                    if (s != u) prod *= (double)B[(int64_t)p[s] * R + r];
                C[(int64_t)p[u] * R + r] += prod;
            }
        }
    }
    return 0;
}

/*
 * Sampled-row oracle: the same expansion, keeping only the permutations whose
 * p_0 is one of rows[0..nrows) (distinct, each in [0,dim)).  C and S are
 * [nrows][R] fp64, overwritten.  Used to check full-size runs row by row.
 */
int oracle_mttkrp_rows(int order, int64_t dim, int64_t nnz, const int32_t *idx,
                       const float *vals, const float *B, int R, int64_t nrows,
                       const int64_t *rows, double *C, double *S, int nthreads) {
    int rc = check_args(order, dim, nnz, idx, vals, B, R);
    if (rc) return rc;
    if (nrows < 0 || (nrows > 0 && (!rows || !C || !S))) return 1;
    int32_t *slot = (int32_t *)malloc((size_t)dim * sizeof(int32_t));
    if (!slot) return 5;
    for (int64_t i = 0; i < dim; i++) slot[i] = -1;
    for (int64_t q = 0; q < nrows; q++) {
        if (rows[q] < 0 || rows[q] >= dim || slot[rows[q]] >= 0) { free(slot); return 1; }
        slot[rows[q]] = (int32_t)q;
    }
    int T = nthreads > 0 ? nthreads : 1;
    const int64_t plane = nrows * (int64_t)R;
    job_t *jobs = (job_t *)calloc((size_t)T, sizeof(job_t));
    double *scratch = (double *)calloc((size_t)T * R, sizeof(double));
    double *priv = (double *)calloc((size_t)T * (plane > 0 ? plane : 1) * 2, sizeof(double));
    if (!jobs || !scratch || !priv) { free(slot); free(jobs); free(scratch); free(priv); return 5; }
    for (int k = 0; k < T; k++) {
        job_t *J = &jobs[k];
        J->order = order; J->dim = dim; J->R = R; J->idx = idx; J->vals = vals; J->B = B;
        J->term = scratch + (int64_t)k * R;
        J->rowslot = slot;
        J->e_begin = nnz * k / T; J->e_end = nnz * (k + 1) / T;
        J->C = priv + (int64_t)k * plane * 2; J->S = J->C + plane;
    }
    run_all(jobs, T);
    memset(C, 0, (size_t)plane * sizeof(double));
    memset(S, 0, (size_t)plane * sizeof(double));
    for (int k = 0; k < T; k++) {
        const double *pc = priv + (int64_t)k * plane * 2, *ps = pc + plane;
        for (int64_t q = 0; q < plane; q++) { C[q] += pc[q]; S[q] += ps[q]; }
    }
    free(slot); free(jobs); free(scratch); free(priv);
    return 0;
}

/* Number of expanded (non-symmetric) updates the oracle performs: the sum of
 * orbit sizes n!/prod m_r!, counted by walking the same permutations. */
int64_t oracle_count_expanded(int order, int64_t nnz, const int32_t *idx) {
    if (order < 1 || order > ORACLE_MAX_ORDER || nnz < 0 || (nnz > 0 && !idx)) return -1;
    int32_t p[ORACLE_MAX_ORDER];
    int64_t count = 0;
    for (int64_t e = 0; e < nnz; e++) {
        for (int t = 0; t < order; t++) p[t] = idx[e * order + t];
        sort_small(p, order);
        do { count++; } while (next_perm(p, order));
    }
    return count;
}

/*
 * General (non-symmetric) sparse MTTKRP, the naive kernel the paper compares
 * against (MTTKRP definitions):
 *   C[idx_e[0], r] += v_e * prod_{t>=1} B[idx_e[t], r],   S likewise with |.|.
 * Tuples are used exactly as given (no canonicalisation, no expansion).
 * Single-threaded: used on small inputs by the NEXT-1 parity tests.
 */
int oracle_mttkrp_general(int order, int64_t dim, int64_t nnz, const int32_t *idx, const float *vals,
                          const float *B, int R, double *C, double *S) {
    int rc = check_args(order, dim, nnz, idx, vals, B, R);
    if (rc) return rc;
    if (!C || !S) return 1;
    memset(C, 0, (size_t)dim * R * sizeof(double));
    memset(S, 0, (size_t)dim * R * sizeof(double));
    for (int64_t e = 0; e < nnz; e++) {
        const int32_t *x = idx + e * order;
        for (int r = 0; r < R; r++) {
            double term = (double)vals[e];
            for (int t = 1; t < order; t++) term *= (double)B[(int64_t)x[t] * R + r];
            C[(int64_t)x[0] * R + r] += term;
            S[(int64_t)x[0] * R + r] += fabs(term);
        }
    }
    return 0;
}

/*
 * One Bellman-Ford relaxation over a symmetric sparse matrix in the (min, +)
 * semiring: every stored entry (a, b, v) stands for both
 * A[a,b] and A[b,a] (Def. Symmetry); the naive kernel visits
 * both orientations (once when a == b):
 *     y[i] = min(d[i], min over expanded (i, j, v) of v + d[j]),
 * each candidate computed as ONE fp32 addition (the precision the GPU path
 * uses, so the min takes the same decision), the min exact.
 */
int oracle_minplus_sym2(int64_t dim, int64_t nnz, const int32_t *idx, const float *vals,
                        const float *d, float *y) {
    if (dim < 1 || nnz < 0 || !d || !y || (nnz > 0 && (!idx || !vals))) return 1;
    for (int64_t k = 0; k < 2 * nnz; k++)
        if (idx[k] < 0 || idx[k] >= dim) return 3;
    for (int64_t i = 0; i < dim; i++) y[i] = d[i];
    for (int64_t e = 0; e < nnz; e++) {
        const int32_t a = idx[2 * e], b = idx[2 * e + 1];
        volatile float cand = vals[e] + d[b];           /* (a, b) orientation */
        if (cand < y[a]) y[a] = cand;
        if (a != b) {                                    /* (b, a) orientation */
            volatile float cand2 = vals[e] + d[a];
            if (cand2 < y[b]) y[b] = cand2;
        }
    }
    return 0;
}

/*
 * Naive TTM on the expanded order-3 tensor:
 *   C[i, j, l] = sum_k A[k, j, l] B[k, i]
 * every distinct permutation (p0, p1, p2) of every stored canonical entry
 * adds v * B[p0, r] to C[p1][p2][r].  C is the FULL output [dim][dim][R] fp64.
 */
int oracle_ttm_sym3(int64_t dim, int64_t nnz, const int32_t *idx, const float *vals, const float *B, int R,
                    double *C) {
    int rc = check_args(3, dim, nnz, idx, vals, B, R);
    if (rc) return rc;
    if (!C) return 1;
    memset(C, 0, (size_t)dim * dim * R * sizeof(double));
    int32_t p[3];
    for (int64_t e = 0; e < nnz; e++) {
        for (int t = 0; t < 3; t++) p[t] = idx[e * 3 + t];
        sort_small(p, 3);
        const double v = (double)vals[e];
        do {
            double *c = C + ((int64_t)p[1] * dim + p[2]) * R;
            const float *b = B + (int64_t)p[0] * R;
            for (int r = 0; r < R; r++) c[r] += v * (double)b[r];
        } while (next_perm(p, 3));
    }
    return 0;
}
