/*
 * systec.h — C ABI of the B200-native symmetric sparse MTTKRP
 * (the hot path of SySTeC, arXiv 2406.09266).
 *
 * The operation ("The assignments for the 3-, 4-, and
 * 5-dimensional kernels"):
 *
 *     C[i, r] = sum_{j_1..j_{n-1}} A[i, j_1, .., j_{n-1}] * prod_t B[j_t, r]
 *
 * where A is a FULLY SYMMETRIC order-n sparse tensor (Def. Symmetry,
 * PAPER.md:141-147) given by its stored entries.  Every stored entry
 * (idx_e, v_e) stands for its whole orbit: A[x] = sum of v_e over the stored
 * entries with sort(x) == sort(idx_e).  Tuples may be given in any order
 * inside the tuple (they are canonicalised, Def. Canonical PAPER.md:162-167,
 * by sorting ascending) and entries in any order; repeated canonical
 * coordinates add (MTTKRP is linear in A).  Each stored entry is read once and
 * updates each of its DISTINCT index positions once, weighted by the number of
 * distinct permutations that put that index first (the unique symmetry group
 * S_P|E, after distributive grouping PAPER.md:577-591).
 *
 * Conventions shared by every entry point
 *   - all array pointers are DEVICE pointers unless the name says _host;
 *   - every device call is ordered on `stream` (0 = legacy default stream);
 *   - indices are 0-based (the paper's Julia listings are 1-based);
 *   - row-major layouts: idx[nnz][order] int32, B[dim][R] fp32, C[dim][R] fp32;
 *   - the caller owns idx, vals, B and C; the library never frees them and
 *     never writes idx, vals or B;
 *   - nothing throws across the ABI: every call returns a systec_status, and
 *     systec_last_cuda_error() gives the cudaError_t behind SYSTEC_ERR_CUDA;
 *   - on an argument error (SYSTEC_ERR_ARG / _UNSUPPORTED / _ALIAS) C is not
 *     touched.
 *   - supported: order 2..5 (3, 4, 5 are the paper's MTTKRP; 2 is symmetric
 *     SpMM), 1 <= dim < 2^31, 0 <= nnz < 2^31, R >= 1, and
 *     order * ceil(log2 dim) <= 64 (one 64-bit sort key).  R % 4 == 0 with
 *     16-byte aligned B and C takes the float4 path; any other R takes the
 *     scalar GPU path (never a CPU path).
 */
#ifndef SYSTEC_H
#define SYSTEC_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define SYSTEC_API __attribute__((visibility("default")))
#else
#define SYSTEC_API
#endif

typedef struct CUstream_st *systec_stream_t;   /* == cudaStream_t */

typedef enum {
    SYSTEC_OK = 0,
    SYSTEC_ERR_ARG = 1,          /* null pointer with nnz>0, dim<1, nnz<0, R<1, bad option   */
    SYSTEC_ERR_UNSUPPORTED = 2,  /* order outside 2..5, dim >= 2^31, nnz >= 2^31 - 64 */
    SYSTEC_ERR_INDEX = 3,        /* some idx outside [0, dim) (detected on the device)      */
    SYSTEC_ERR_ALIAS = 4,        /* C overlaps B, idx or vals                               */
    SYSTEC_ERR_NOMEM = 5,        /* device or host allocation failed                        */
    SYSTEC_ERR_CUDA = 6          /* a CUDA runtime call failed; see systec_last_cuda_error  */
} systec_status;

/* Statistics of a prepared plan (filled once, at plan creation). */
typedef struct systec_stats {
    int64_t nnz;                 /* stored entries                                            */
    int64_t dim;
    int32_t order;
    int32_t key_bits;            /* bits per index in the sort key = ceil(log2 dim); order*key_bits > 64: a wide plan */
    int64_t G;                   /* sum over entries of the number of distinct indices d_e     */
    int64_t expanded;            /* sum over entries of the orbit size n!/prod m! (naive work) */
    int64_t pattern_hist[16];    /* entries per equality-pattern code (bit t: c_t == c_{t+1})  */
    int64_t lead_runs;           /* runs of equal leading index c_0 in the plan's stream order */
    int64_t max_lead_run;        /* longest such run                                           */
    int64_t pos1_runs;           /* runs of equal c_1 in the plan's stream order               */
    int32_t input_was_sorted;    /* 1: input already canonical and lexicographically sorted    */
    int32_t band_shift;          /* -1: stream in lexicographic order; s >= 0: grouped by band */
                                 /* c_{n-1} >> s, lexicographic within a band (plan options)   */
    int64_t bad_entry;           /* first entry with an index outside [0,dim), else -1         */
    int64_t bandwidth;           /* order 2: max (c_1 - c_0) over entries; else 0              */
    int64_t window_blocks;       /* order 2: row blocks of the atomic-free windowed kernel     */
                                 /* (0 = the plan runs the general kernel; see execute opts)   */
} systec_stats;

/* Kernel tuning options for systec_plan_execute_ex; zero fields = defaults. */
typedef struct systec_exec_opts {
    int32_t warps_per_block;     /* 0 = default (8)                                            */
    int32_t blocks_per_sm;       /* 0 = as many as fit (occupancy calculator)                  */
    int32_t pos1_accumulate;     /* 0 = auto from stats, 1 = on, -1 = off                      */
    int32_t force_scalar;        /* 1 = scalar (non-float4) path even when float4 is possible  */
    int32_t no_zero;             /* 1 = accumulate into C instead of overwriting it            */
    int32_t l2_hints;            /* 0 = default (on), -1 = off                                 */
    int32_t chunk_k;             /* entries per lane group per staged chunk (0 = auto)         */
    int32_t stages;              /* shared-memory ring depth of the stream staging (0 = 2)     */
    int32_t vpl;                 /* float4 per lane: 1, 2 or 4 (0 = 1)                          */
    int32_t prefetch;            /* next entry's B rows in flight: 1 on, 0/-1 off              */
    int32_t copies;              /* replicas of C for L2-slice spreading: 1 = off, 0 = auto     */
                                 /* (auto: C < 4 MB and nnz >= 1e5 -> up to 32 replicas)        */
    int32_t ablation;            /* evidence study, c2/c5 kernel shapes only: bit 0 = no smem  */
                                 /* staging of the stream, bit 1 = no position-0 accumulation  */
    int32_t static_ranges;       /* 1 = one static nnz-balanced range per warp; 0 = dynamic units */
                                 /* of ~4 chunks taken from a per-launch counter (default)       */
    int32_t occupancy;           /* order-3 R=32 kernel built for 5 blocks/SM: 1 on, -1 off,    */
                                 /* 0 auto (on when B > 64 MB and the plan is lexicographic)   */
    int32_t fixed_rank;          /* kernels built for R = 16 / 32 exactly (one float4 tile):    */
                                 /* 0 auto (on when R matches; general plans: off), 1 on, -1 off */
    int32_t window;              /* order-2 plans created with systec_plan_opts.window = 1: the */
                                 /* atomic-free windowed kernel (each row block builds its     */
                                 /* rows' transposed entries in shared memory and writes every */
                                 /* output row once): 0 auto (on when stats.window_blocks > 0), */
                                 /* -1 off                                                      */
    int32_t lane_bytes;          /* columns per lane of the fixed-rank builds: 16 (4 floats,   */
                                 /* 128-bit gathers) or 32 (8 floats, 256-bit gathers, R = 16 */
                                 /* / 32 with 32-byte aligned B and C); 0 = auto              */
} systec_exec_opts;

typedef struct systec_plan_s *systec_plan;

/* Plan-creation options for systec_plan_create_ex; zero fields = defaults. */
typedef struct systec_plan_opts {
    int32_t band_shift;          /* stream order: 0 = auto, -1 = lexicographic, s > 0 = group  */
                                 /* entries by band c_{n-1} >> s (band-major, lexicographic    */
                                 /* within a band; at most 2^16 bands, else lexicographic)     */
                                 /* by one stable radix pass over the band numbers.  Auto bands */
                                 /* order-3 plans with dim >= 2^19 into up to 16 bands (no     */
                                 /* fewer than 2^16 rows each; fewer bands when leading runs   */
                                 /* are short): the rows that positions >= 1 gather and update */
                                 /* then stay within an L2-sized window while a band runs.     */
                                 /* Any order gives the same C up to fp32 rounding order.      */
                                 /* General plans are banded only on request (explicit s).     */
    int32_t general;             /* 1 = a general (non-symmetric) tensor, as                   */
                                 /* systec_plan_create_general; 0 = symmetric                  */
    int32_t window;              /* order-2 symmetric plans: 1 = also build the row / column   */
                                 /* pointers of the atomic-free windowed kernel (used when the */
                                 /* bandwidth is small; measured slower than the default       */
                                 /* kernel on the banded stand-in); 0 = no      */
    int32_t reserved[5];
} systec_plan_opts;

/*
 * One-shot call with the paper's signature (north_star):
 * plan_create + plan_execute + plan_destroy.  idx/vals/B/C are DEVICE
 * pointers; C [dim][R] is OVERWRITTEN.  Synchronises `stream` inside plan
 * creation (validation verdict and statistics); the execute part is async.
 * The plan is used once, so it keeps the lexicographic stream order (no band
 * re-sort, systec_plan_opts).
 */
SYSTEC_API int systec_mttkrp(int order, int64_t dim, int64_t nnz, const int32_t *idx, const float *vals,
                  const float *B, int R, float *C, systec_stream_t stream);

/*
 * The same operation on HOST buffers (the end-to-end call): copies idx, vals
 * and B to the device, runs the path, copies C back and synchronises.
 * Host buffers may be pageable or pinned (pinned is faster).  Device scratch
 * comes from the stream-ordered pool and is returned before the call ends.
 * The input is processed in chunks whose copies overlap the previous chunk's
 * work; with page-locked C, rows no later chunk can touch are copied back
 * early.  Errors: on SYSTEC_ERR_INDEX (an index outside [0, dim) in any
 * chunk; systec_last_bad_entry() names the first one) C_host holds no valid
 * result — rows copied back before the bad chunk was seen may already have
 * been overwritten with partial sums, and the chunks were processed with
 * the offending coordinates clamped — so treat all of C_host as garbage.
 * On argument errors (SYSTEC_ERR_ARG / _UNSUPPORTED / _ALIAS) C_host is
 * untouched.
 */
SYSTEC_API int systec_mttkrp_host(int order, int64_t dim, int64_t nnz, const int32_t *idx_host,
                       const float *vals_host, const float *B_host, int R, float *C_host,
                       systec_stream_t stream);

/*
 * Plan creation: validate (range check on the device), canonicalise every
 * tuple (ascending sort), sort entries lexicographically (skipped when the
 * input already is), and store the prepared structure-of-arrays copy
 * (order x int32 + 1 x fp32 per entry, owned by the plan).  idx and vals may
 * be freed once this returns.  The plan belongs to the device current at
 * creation; execute it there.  Input already in storage order (canonical
 * forms sorted lexicographically) is prepared in one device pass —
 * validation, the structure-of-arrays copy, the sortedness verdict and the
 * statistics — and ONE synchronisation of `stream`; any other order takes the
 * sorting path after that verdict and synchronises once more to read the
 * statistics of the sorted stream.
 * Errors: ARG, UNSUPPORTED, INDEX (plan not created, *out = NULL, and
 * systec_last_bad_entry() names the first offending entry), NOMEM, CUDA.
 */
SYSTEC_API int systec_plan_create(systec_plan *out, int order, int64_t dim, int64_t nnz,
                       const int32_t *idx, const float *vals, systec_stream_t stream);

/*
 * systec_plan_create with options (NULL = defaults, i.e. systec_plan_create).
 * A banded plan (systec_plan_opts.band_shift) re-sorts its prepared stream
 * once more on the device (one more synchronisation of `stream`).
 * Errors: as systec_plan_create; ARG for band_shift < -1, general not 0/1 or
 * a non-zero reserved field.
 */
SYSTEC_API int systec_plan_create_ex(systec_plan *out, int order, int64_t dim, int64_t nnz,
                                     const int32_t *idx, const float *vals, const systec_plan_opts *opts,
                                     systec_stream_t stream);

/*
 * The non-symmetric baseline (the paper's "naive"
 * kernels): a plan over a GENERAL sparse tensor —
 * tuples are validated and sorted lexicographically but NOT canonicalised —
 * whose execute computes C[i,r] = sum_{e: idx_e[0] = i} v_e prod_{t>=1} B[idx_e[t], r]
 * (one update per stored entry, leading-index runs accumulated in registers).
 * Fed with systec_expand_symmetric's output it computes the same C as the
 * symmetric plan, doing the work the symmetric method avoids.  Same
 * arguments, errors and ownership as systec_plan_create.
 */
SYSTEC_API int systec_plan_create_general(systec_plan *out, int order, int64_t dim, int64_t nnz,
                                          const int32_t *idx, const float *vals, systec_stream_t stream);

/*
 * One Bellman-Ford relaxation in the (min, +) semiring over a symmetric sparse
 * MATRIX (an order-2 plan, the paper's Bellman-Ford
 * kernel `y[i] min= A[i,j] + d[j]`):
 *     y[i] = min(d[i], min over stored (i,j,v) or (j,i,v) of v + d[j])
 * d [dim] and y [dim] are device fp32 vectors (must not overlap).  Each
 * candidate is one fp32 add and the min is exact, so the result does not
 * depend on the update order.  Async on `stream`.
 * Errors: ARG, UNSUPPORTED (plan order != 2 or a general plan), ALIAS, CUDA.
 */
SYSTEC_API int systec_plan_minplus(systec_plan plan, const float *d, float *y, systec_stream_t stream);

/*
 * Symmetric CP decomposition by alternating least squares (SURVEY.md §8(f)
 * NEXT-2; one factor matrix for every mode, so the update is
 * the same in all modes).  X ≈ sum_r lambda_r b_r^{(x)n}.  Each iteration:
 *     M = MTTKRP(X, B);  B = M ((B^T B)^{.(n-1)})^{-1};  lambda = column norms;  B /= lambda
 * (R = 1 is the symmetric higher-order power method).  B [dim][R] (device) holds
 * the initial factor on entry and the unit-column factor on return; lambda [R]
 * (device) receives the weights (max_iters = 0: B is returned unchanged and
 * lambda = 1).  Runs up to max_iters iterations and stops
 * early when the fit changes by less than tol; fit_host [max_iters] (host, may
 * be NULL) receives fit_k = 1 - ||X - Xhat_k|| / ||X|| of each iterate;
 * *iters_done the number of iterations run.  1 <= R <= 48.  For runs of
 * max_iters >= 16 the iteration loop is device-resident: one CUDA graph whose
 * conditional WHILE node repeats the dense pass -> (the fit, the R x R update
 * and a device convergence test, beside the next MTTKRP), synchronising
 * `stream` once at the end; shorter runs use a host loop
 * that synchronises once per iteration to read the fit (the graph costs
 * ~0.4 ms to build).  Environment SYSTEC_CPALS_LOOP=host|graph overrides.
 * Errors: ARG, UNSUPPORTED (general plan, R > 48), ALIAS, NOMEM, CUDA.
 */
SYSTEC_API int systec_cp_als_sym(systec_plan plan, float *B, int R, float *lambda, int max_iters, double tol,
                                 double *fit_host, int *iters_done, systec_stream_t stream);

/*
 * Testing entry point: ONE CP-ALS dense pass at R = 32 — the iteration's only
 * dim x R pass (PAPER.md:853-857 for the update; reading X25 for the
 * one-pass form) — in a chosen kernel form, so that the tensor-core forms can
 * be checked against a reference and against each other:
 *   form 0: legacy mma.sync (m16n8k8 TF32) 3xTF32 kernel;
 *   form 1: tcgen05.mma kind::tf32 3xTF32 kernel, accumulators in TMEM.
 * M, F: [dim][32] device fp32, 16-byte aligned; W: [32][32] device fp32.
 * part: device fp64, room for 1024 blocks of (32*32 + 32): block b receives
 * {sum over its rows of M^T M (row-major 32 x 32), sum over its rows of M o F
 * (32 column dots)}; the sums over the returned number of blocks are the pass's
 * totals.  store != 0: F is overwritten with M W after its dots are taken.
 * Async on `stream`.  Returns the number of blocks written (>= 1), or
 * -SYSTEC_ERR_ARG / -SYSTEC_ERR_UNSUPPORTED (form not available: misaligned,
 * or no tensor-map encoder) / -SYSTEC_ERR_CUDA.
 */
SYSTEC_API int systec_testing_cpd_pass(int form, int64_t dim, const float *M, float *F, const float *W, double *part,
                                       int store, systec_stream_t stream);

/*
 * Single-source shortest paths by Bellman-Ford over a symmetric sparse matrix
 * of edge weights (an order-2 plan: stored (i, j, w) is the undirected edge
 * i-j): dist [dim] (device, out) starts at +inf except dist[source] = 0 and is
 * relaxed with systec_plan_minplus until no entry changes or max_iters
 * relaxations ran; *iters_done (may be NULL) receives the relaxations done,
 * counting the last one that changed nothing.  Weights must not create
 * negative cycles (an undirected negative edge is one).  Synchronises `stream`
 * once per iteration (environment SYSTEC_SSSP_LOOP=graph: the loop runs on the
 * device as one CUDA graph with a conditional WHILE node, one synchronisation
 * at the end — for graphs needing many relaxations).
 * Errors: ARG, UNSUPPORTED (order != 2), NOMEM, CUDA.
 */
SYSTEC_API int systec_plan_sssp(systec_plan plan, int64_t source, float *dist, int max_iters, int *iters_done,
                                systec_stream_t stream);

/*
 * Symmetric TTM with visible output symmetry (the
 * paper's TTM, Listings 1-3 PAPER.md:262-325), order-3 plans:
 *     C[i, j, l] = sum_k A[k, j, l] B[k, i],    C[i,j,l] = C[i,l,j]
 * Only the canonical half j <= l is computed, packed as
 * C_packed [dim(dim+1)/2][R] (device; row pair(j,l) = l(l+1)/2 + j, rank
 * innermost), OVERWRITTEN.  B [dim][R] device.  Async on `stream`.
 * On a GENERAL order-3 plan (the naive baseline, e.g. over the expanded
 * tensor) the LAST mode is contracted — C[p0][p1][:] += v B[p2][:], the mode
 * innermost in the sorted stream, so runs of equal (p0, p1) accumulate in
 * registers — and C_packed must hold the full [dim][dim][R] tensor instead
 * (for the expansion of a symmetric tensor: the same C as above).
 * Errors: ARG, UNSUPPORTED (order != 3), ALIAS, CUDA.
 */
SYSTEC_API int systec_plan_ttm(systec_plan plan, const float *B, int R, float *C_packed, systec_stream_t stream);

/*
 * Replicate the packed TTM output to the full tensor C_full [dim][dim][R]
 * (device; C_full[j][l][i] = C[i,j,l]) — the output replication the paper
 * excludes from its timings.  Async.  Errors: ARG, ALIAS, CUDA.
 */
SYSTEC_API int systec_ttm_unpack(int64_t dim, int R, const float *C_packed, float *C_full, systec_stream_t stream);

/*
 * Expand a symmetric tensor's stored entries (device idx [nnz][order], vals
 * [nnz]; any tuple order) into every distinct permutation of each tuple — the
 * non-symmetric tensor it stands for (Def. Symmetry, PAPER.md:141-147;
 * n!/prod m! members per entry).  *count receives the total.
 * out_idx == out_vals == NULL: count only.  Otherwise out_idx [capacity][order]
 * and out_vals [capacity] (device) receive the entries, grouped by input
 * entry, each group in lexicographic order; capacity < *count -> ERR_ARG.
 * Synchronises `stream` once.  Errors: ARG, UNSUPPORTED, INDEX, NOMEM, CUDA.
 */
SYSTEC_API int systec_expand_symmetric(int order, int64_t dim, int64_t nnz, const int32_t *idx,
                                       const float *vals, int64_t capacity, int32_t *out_idx,
                                       float *out_vals, int64_t *count, systec_stream_t stream);

/*
 * Execute: C[dim][R] = MTTKRP(plan, B).  Zeroes C and launches the kernel on
 * `stream`; never synchronises (CUDA-graph capturable).  Its only allocation
 * is stream-ordered scratch from the device's default pool (cudaMallocAsync)
 * for the replicas of a small C (< 4 MB), returned before the call's work ends.
 * Concurrent executions of one plan on different streams are safe when
 * their C buffers differ.  Errors: ARG, ALIAS, CUDA (launch failure).
 */
SYSTEC_API int systec_plan_execute(systec_plan plan, const float *B, int R, float *C, systec_stream_t stream);

/* Execute with tuning options (NULL = defaults).  Same semantics. */
SYSTEC_API int systec_plan_execute_ex(systec_plan plan, const float *B, int R, float *C,
                           const systec_exec_opts *opts, systec_stream_t stream);

/* Copy the plan's statistics to host memory. */
SYSTEC_API int systec_plan_stats(systec_plan plan, systec_stats *host_out);

/*
 * Device pointers to the prepared stream (read-only views, owned by the plan):
 * coords[t] = c_t[nnz] int32 for t < order, *vals = v[nnz] fp32, in
 * lexicographic order of the canonical tuples.  For tests and tools.
 */
SYSTEC_API int systec_plan_prepared(systec_plan plan, const int32_t **coords /* [order] */, const float **vals);

/* Copy the prepared stream into caller-owned DEVICE buffers, ordered on
 * `stream`: coords_dst [order][nnz] int32 (row t = c_t), vals_dst [nnz] fp32. */
SYSTEC_API int systec_plan_copy_prepared(systec_plan plan, int32_t *coords_dst, float *vals_dst,
                                         systec_stream_t stream);

/* Launch geometry of the last execute of this plan (for bench reporting). */
SYSTEC_API int systec_plan_last_launch(systec_plan plan, int32_t *grid_x, int32_t *grid_y, int32_t *block,
                            int32_t *smem_bytes, int32_t *kernel_id);

/* Free the plan's device memory (stream-ordered on the creation stream). */
SYSTEC_API int systec_plan_destroy(systec_plan plan);

SYSTEC_API const char *systec_status_string(int status);
SYSTEC_API int systec_last_cuda_error(void);
/* ABI version: 100 * major + minor. */
SYSTEC_API int systec_version(void);
/* Entry index of the first out-of-range tuple seen by the last failed
 * plan creation on this thread (SYSTEC_ERR_INDEX), else -1. */
SYSTEC_API int64_t systec_last_bad_entry(void);

#ifdef __cplusplus
}
#endif
#endif /* SYSTEC_H */
