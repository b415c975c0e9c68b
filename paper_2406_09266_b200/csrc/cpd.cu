// cpd.cu — symmetric CP decomposition by alternating least squares, the
// consumer MTTKRP exists for ("the
// symmetric CPD problem uses the same factor matrix for all dimensions ... the
// update step is identical in all the modes").  The paper does not print the
// update; we use the symmetric ALS step (the one-factor form of CP-ALS, whose
// R = 1 case is the symmetric higher-order power method of the cited Kofidis &
// Regalia): for X ≈ sum_r lambda_r b_r^{(x)n},
//
//     M      = MTTKRP(X, B)                       (the symmetric kernel)
//     H      = (B^T B)^{.(n-1)}                   (Hadamard power, R x R)
//     B_new  = M H^{-1}                           (R x R SPD solve)
//     lambda = column 2-norms of B_new,  B = B_new / lambda.
//
// Fit of the iterate (B, lambda), computed from the NEXT iteration's M (no extra
// MTTKRP):  <X, Xhat> = sum_r lambda_r sum_i M[i,r] B[i,r],
//           ||Xhat||^2 = lambda^T (B^T B)^{.n} lambda,
//           ||X||^2   = sum_e v_e^2 * orbit_e   (each stored entry stands for its orbit),
//           fit = 1 - sqrt(max(0, ||X||^2 - 2<X,Xhat> + ||Xhat||^2)) / ||X||.
//
// Dense work per iteration (after the MTTKRP): ONE row pass over the dim x R
// matrices, the normalisation folded into the R x R algebra.  Two facts make
// that possible:
//   * B_new^T B_new = H^{-1} G_M H^{-1} for B_new = M H^{-1} (H symmetric), so
//     the new lambda and the next G_B follow from G_M = M^T M alone;
//   * MTTKRP is multilinear, MTTKRP(X, B diag(t)) = MTTKRP(X, B) diag(t)^{n-1},
//     so the stored factor F may carry any known column scale t.
// The pass reads M and F once: it accumulates G_M and the dots M o F (the
// fit of the current iterate) and writes F_new = M W with W = diag(t)^{-(n-1)}
// H^{-1} diag(1/lambda) — the current lambda predicts the new one, so F_new =
// B_new diag(lambda_new / lambda) stays near unit columns.  The small solve
// (one block, fp64, cp_small_kernel) then takes the exact new lambda and t from
// diag(W^T G_M W) and builds the next W.  At R = 32 the pass is one fused
// tensor-core kernel (pass_tc32_kernel); other ranks run it as a Gram/dots
// launch and an apply launch.  Iteration 0 (the caller's factor, arbitrary
// scale) runs the Gram first and writes B_1 normalised; the call ends with one
// F /= t pass.  (Round 1: Gram of B, apply, column norms, normalise — four
// passes; round 2 before this: Gram of M + apply — two.)  The first
// iteration's G_B is one Gram pass over the caller's B.
//
// Every step runs in the kernels below (R <= 48; the small R x R algebra in
// one block, in fp64).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#ifdef SYSTEC_EXP_SMALL_CLOCKS
#include <cstdio>
#endif

#include "internal.cuh"
#include "ptx.cuh"

namespace systec {

namespace {

constexpr int kMaxCpR = 48;  // [R][2R] fp64 Gauss-Jordan tableau (36 KB) in static shared memory

// Two-stage reductions (no global atomics): every block owns a contiguous row
// range and writes fp64 partial sums; reduce_partials_kernel adds the blocks.
//
// gram_dots_partial_kernel: part[blk][a*R+b] = sum_{i in blk} B[i][a] B[i][b]
//                           part[blk][R*R+r] = sum_{i in blk} M[i][r] B[i][r]
// Rows are staged in shared memory in tiles of kTileRows; each thread owns a
// 4x4 register tile of (a, b) pairs for one row group (rows i = g mod RG) and
// accumulates a tile in fp32 before adding it to fp64; the row groups are
// summed in shared memory.  (Reading the rows straight from L1 instead, no
// staging, measured 3x slower.)
#ifndef SYSTEC_CPD_TILE_ROWS
#define SYSTEC_CPD_TILE_ROWS 128
#endif
#ifndef SYSTEC_CPD_RING
#define SYSTEC_CPD_RING 3
#endif
#ifndef SYSTEC_CPD_BPS
#define SYSTEC_CPD_BPS 2
#endif
constexpr int kTileRows = SYSTEC_CPD_TILE_ROWS;
constexpr int kRp = (kMaxCpR + 3) / 4 * 4;  // padded column count (multiple of 4)

// rows [r0, r0+nr) of X[.][R] -> dst[nr][Rp] (zero-padded columns; 16-byte
// loads, all of a thread's loads issued before its stores)
__device__ __forceinline__ void stage_rows(float *__restrict__ dst, const float *__restrict__ X, int64_t r0, int nr,
                                           int R, int Rp) {
    const int tid = threadIdx.x, nt = blockDim.x;
    if (Rp == R) {  // contiguous rows: a 16-byte copy (R % 4 == 0 keeps every row aligned)
        const int n4 = nr * R / 4;
        const float4 *s4 = reinterpret_cast<const float4 *>(X + r0 * R);
        float4 *d4 = reinterpret_cast<float4 *>(dst);
        for (int q = tid; q < n4; q += 4 * nt) {
            float4 v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (q + u * nt < n4) v[u] = __ldg(s4 + q + u * nt);
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (q + u * nt < n4) d4[q + u * nt] = v[u];
        }
    } else {
        for (int q = tid; q < nr * Rp; q += nt) {
            const int i = q / Rp, c = q % Rp;
            dst[q] = c < R ? __ldg(X + (r0 + i) * R + c) : 0.f;
        }
    }
}

// S-stage ring of row tiles [kTileRows][R] of one or two matrices, filled by
// 1-D bulk copies (TMA engine, one per matrix and tile, completing on the
// stage's mbarrier) that thread 0 issues S-1 tiles ahead of the block's
// arithmetic — contiguous rows only (R % 4 == 0, 16-byte aligned bases).
// (Double-buffered per-thread cp.async copies measured Gram 115 us on c3, the
// bulk ring below is what runs now.)
constexpr int kRingS = SYSTEC_CPD_RING;
template <int S>
struct TileRingT {
    float *buf;       // [S][NM][kTileRows * R]
    uint64_t *bars;   // [S]
    const float *X0, *X1;
    int NM, R;
    int64_t lo, hi;
    __device__ int64_t ntiles() const { return (hi - lo + kTileRows - 1) / kTileRows; }
    __device__ float *tile(int64_t k, int m) const {
        return buf + (static_cast<size_t>(k % S) * NM + m) * kTileRows * R;
    }
    __device__ void init() const {  // thread 0, then a block barrier
        for (int st = 0; st < S; ++st) mbar_init(&bars[st], 1);
        fence_mbar_init();
    }
    __device__ void issue(int64_t k) const {  // thread 0
        const int64_t r0 = lo + k * kTileRows;
        const uint32_t bytes = static_cast<uint32_t>(min(static_cast<int64_t>(kTileRows), hi - r0) * R * 4);
        uint64_t *bar = &bars[k % S];
        const uint64_t pol = policy_evict_first();
        mbar_arrive_expect_tx(bar, bytes * NM);
        bulk_g2s(tile(k, 0), X0 + r0 * R, bytes, bar, pol);
        if (NM > 1) bulk_g2s(tile(k, 1), X1 + r0 * R, bytes, bar, pol);
    }
    __device__ void wait(int64_t k) const { mbar_wait(&bars[k % S], static_cast<uint32_t>((k / S) & 1)); }
};
using TileRing = TileRingT<kRingS>;
template <int S = kRingS>
__host__ __device__ constexpr size_t ring_bytes(int NM, int R) {
    return static_cast<size_t>(S) * NM * kTileRows * R * 4 + S * 8;
}

__global__ void __launch_bounds__(256) gram_dots_partial_kernel(const float *__restrict__ B, const float *__restrict__ M,
                                                                int64_t dim, int R, double *__restrict__ part) {
    extern __shared__ __align__(16) unsigned char cpd_smem[];
    // one synchronously staged [kTileRows][Rp] tile of B and of M (general R;
    // R % 4 == 0, R <= 32 runs gram_dots_sym_kernel on the bulk-copy ring)
    float *tbuf = reinterpret_cast<float *>(cpd_smem);
    constexpr int kTile = kTileRows * kRp;
    double *red = reinterpret_cast<double *>(cpd_smem);  // reused after the row loop
    const int Rp = (R + 3) & ~3;
    const int T4 = Rp / 4;           // 4-wide column blocks
    const int MT = T4 * T4;          // micro-tiles
    const int RG = blockDim.x / MT;  // row groups
    const int tid = threadIdx.x;
    const int mt = tid % MT, g = tid / MT;
    const int a0 = (mt / T4) * 4, b0 = (mt % T4) * 4;
    const bool active = g < RG;
    const int64_t rows = (dim + gridDim.x - 1) / gridDim.x;
    const int64_t lo = blockIdx.x * rows, hi = min(dim, lo + rows);
    double acc[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) acc[k] = 0.0;
    double dacc = 0.0;  // column dot: thread (column tid % R, row lane tid / R)
    const int dl = tid / R, dn = blockDim.x / R;
    for (int64_t r0 = lo; r0 < hi; r0 += kTileRows) {
        const int nr = static_cast<int>(min(static_cast<int64_t>(kTileRows), hi - r0));
        float *tb = tbuf, *tm = tbuf + kTile;
        stage_rows(tb, B, r0, nr, R, Rp);
        stage_rows(tm, M, r0, nr, R, Rp);
        __syncthreads();
        if (active) {
            float f[16];
#pragma unroll
            for (int k = 0; k < 16; ++k) f[k] = 0.f;
#pragma unroll 2
            for (int i = g; i < nr; i += RG) {
                const float4 x = *reinterpret_cast<const float4 *>(tb + i * Rp + a0);
                const float4 y = *reinterpret_cast<const float4 *>(tb + i * Rp + b0);
                const float xa[4] = {x.x, x.y, x.z, x.w}, yb[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
                for (int u = 0; u < 4; ++u)
#pragma unroll
                    for (int v = 0; v < 4; ++v) f[u * 4 + v] = fmaf(xa[u], yb[v], f[u * 4 + v]);
            }
#pragma unroll
            for (int k = 0; k < 16; ++k) acc[k] += f[k];
        }
        if (dl < dn) {
            const int c = tid % R;
            float d = 0.f;
            for (int i = dl; i < nr; i += dn) d = fmaf(tm[i * Rp + c], tb[i * Rp + c], d);
            dacc += d;
        }
        __syncthreads();  // tile k consumed: its slot may be refilled
    }
    __syncthreads();  // tiles no longer needed: sum the row groups in shared memory
    double *dred = red + kRp / 4 * (kRp / 4) * 16;  // [256] after the pair sums
    dred[tid] = dl < dn ? dacc : 0.0;
    const int W = R * R + R;
    double *out = part + static_cast<int64_t>(blockIdx.x) * W;
    for (int grp = 0; grp < RG; ++grp) {
        if (active && g == grp) {
#pragma unroll
            for (int k = 0; k < 16; ++k) red[mt * 16 + k] = (grp == 0 ? 0.0 : red[mt * 16 + k]) + acc[k];
        }
        __syncthreads();
    }
    for (int q = tid; q < MT * 16; q += blockDim.x) {
        const int m = q / 16, k = q % 16;
        const int a = (m / T4) * 4 + k / 4, b = (m % T4) * 4 + k % 4;
        if (a < R && b < R) out[a * R + b] = red[q];
    }
    if (tid < R) {
        double d = 0.0;
        for (int l = 0; l < dn; ++l) d += dred[l * R + tid];
        out[R * R + tid] = d;
    }
}

// ---- tensor-core forms (R = 32): 3xTF32 mma.sync ----------------------------
// Both dense passes are contractions over a dim x 32 matrix: pass A's Gram
// M^T M (K = the rows) and pass B's M W (K = 32).  On FFMAs they are bound by
// issue (c3: 41M / 52M warp instructions, 55-62 % issue-active, ncu
// profiles/r02/cpd_c3_ncu_raw.csv); as m16n8k8 TF32 tensor-core MMAs they need a
// tenth of the instructions.  fp32 accuracy is kept by the 3xTF32 split: x =
// x_hi + x_lo with x_hi = tf32(x), x_lo = tf32(x - x_hi), and
// a b ~ a_hi b_hi + a_hi b_lo + a_lo b_hi (relative error ~2^-21 per
// product, fp32 accumulation inside the MMA, fp64 across tiles).
__device__ __forceinline__ uint32_t tf32_of(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ void split_tf32(float x, uint32_t &hi, uint32_t &lo) {
    hi = tf32_of(x);
    lo = tf32_of(x - __uint_as_float(hi));
}
// D (16x8, fp32) += A (16x8, tf32, row) * B (8x8, tf32, col)
__device__ __forceinline__ void mma_tf32(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                 "{%0,%1,%2,%3};"
                 : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void mma3(float (&d)[4], const uint32_t (&ah)[4], const uint32_t (&al)[4], uint32_t bh0,
                                     uint32_t bh1, uint32_t bl0, uint32_t bl1) {
#ifndef SYSTEC_EXP_1XTF32  // experiment builds only: one MMA (accuracy lost) to time the MMA share
    mma_tf32(d, al, bh0, bh1);  // small terms first
    mma_tf32(d, ah, bl0, bl1);
#endif
    mma_tf32(d, ah, bh0, bh1);
}

// Pass A at R = 32 on tensor cores: part[blk] = {M^T M (32 x 32), dots M o B}.
// Warp w takes rows [16w, 16w+16) of each 128-row tile (two K steps of 8
// rows).  The output columns are permuted so that one LDS.128 gives a thread
// all its fragments: logical column n = 8 nt + g lives at physical column
// 4 g + nt, so thread (g = lane/4, t = lane%4) reads physical columns 4g..4g+3
// of rows t and t+4 — the B fragments of the four n-tiles — and, the Gram
// being M^T M, the A fragments of m-tile mb are the B fragments of n-tiles
// 2mb and 2mb+1.  Only the upper block triangle is computed (6 of 8 16x8
// tiles) and mirrored.  The column dots use float4 lanes as the FFMA form.
__global__ void __launch_bounds__(256) gram_tc32_kernel(const float *__restrict__ X, const float *__restrict__ Y,
                                                        int64_t dim, double *__restrict__ part) {
    constexpr int R = 32;
    extern __shared__ __align__(16) unsigned char cpd_smem[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
    const int cq = tid % 8, rl = tid / 8, nrl = blockDim.x / 8;  // column dots: (row lane, float4 column)
    const int64_t rows = (dim + gridDim.x - 1) / gridDim.x;
    const int64_t lo = blockIdx.x * rows, hi = min(dim, lo + rows);
    TileRing tr{reinterpret_cast<float *>(cpd_smem), reinterpret_cast<uint64_t *>(cpd_smem + ring_bytes(2, R) - kRingS * 8),
                X, Y, 2, R, lo, hi};
    const int64_t nt = lo < hi ? tr.ntiles() : 0;
    if (tid == 0) {
        tr.init();
        for (int64_t q = 0; q < min(static_cast<int64_t>(kRingS - 1), nt); ++q) tr.issue(q);
    }
    __syncthreads();
    // output tiles: (mb, nb) = (0,0) (0,1) (0,2) (0,3) (1,2) (1,3)
    constexpr int kTiles = 6;
    double acc[kTiles][4];
#pragma unroll
    for (int q = 0; q < kTiles; ++q)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[q][e] = 0.0;
    double dacc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int64_t k = 0; k < nt; ++k) {
        const int nr = static_cast<int>(min(static_cast<int64_t>(kTileRows), hi - lo - k * kTileRows));
        if (tid == 0 && k + kRingS - 1 < nt) {
            fence_proxy_async_smem();
            tr.issue(k + kRingS - 1);
        }
        const float *tx = tr.tile(k, 0), *ty = tr.tile(k, 1);
        tr.wait(k);
        for (int w0 = warp * 16; w0 < nr; w0 += 8 * 16) {  // (kTileRows 128: one slab per warp)
            float f[kTiles][4];
#pragma unroll
            for (int q = 0; q < kTiles; ++q)
#pragma unroll
                for (int e = 0; e < 4; ++e) f[q][e] = 0.f;
#pragma unroll
            for (int ks = 0; ks < 2; ++ks) {
                const int r0 = w0 + ks * 8 + t, r1 = r0 + 4;  // rows past nr are zero-weighted below
                const float4 v0 = r0 < nr ? *reinterpret_cast<const float4 *>(tx + r0 * R + 4 * g) : make_float4(0.f, 0.f, 0.f, 0.f);
                const float4 v1 = r1 < nr ? *reinterpret_cast<const float4 *>(tx + r1 * R + 4 * g) : make_float4(0.f, 0.f, 0.f, 0.f);
                uint32_t bh[4][2], bl[4][2];  // [n-tile][b0 / b1]
                split_tf32(v0.x, bh[0][0], bl[0][0]); split_tf32(v1.x, bh[0][1], bl[0][1]);
                split_tf32(v0.y, bh[1][0], bl[1][0]); split_tf32(v1.y, bh[1][1], bl[1][1]);
                split_tf32(v0.z, bh[2][0], bl[2][0]); split_tf32(v1.z, bh[2][1], bl[2][1]);
                split_tf32(v0.w, bh[3][0], bl[3][0]); split_tf32(v1.w, bh[3][1], bl[3][1]);
#pragma unroll
                for (int mb = 0; mb < 2; ++mb) {
                    const uint32_t ah[4] = {bh[2 * mb][0], bh[2 * mb + 1][0], bh[2 * mb][1], bh[2 * mb + 1][1]};
                    const uint32_t al[4] = {bl[2 * mb][0], bl[2 * mb + 1][0], bl[2 * mb][1], bl[2 * mb + 1][1]};
#pragma unroll
                    for (int nb = 2 * mb; nb < 4; ++nb) {
                        const int q = mb == 0 ? nb : 2 + nb;  // (1,2) -> 4, (1,3) -> 5
                        mma3(f[q], ah, al, bh[nb][0], bh[nb][1], bl[nb][0], bl[nb][1]);
                    }
                }
            }
#pragma unroll
            for (int q = 0; q < kTiles; ++q)
#pragma unroll
                for (int e = 0; e < 4; ++e) acc[q][e] += f[q][e];
        }
        if (rl < nrl) {
            float4 d = make_float4(0.f, 0.f, 0.f, 0.f);
            for (int i = rl; i < nr; i += nrl) {
                const float4 x4 = *reinterpret_cast<const float4 *>(tx + i * R + 4 * cq);
                const float4 y4 = *reinterpret_cast<const float4 *>(ty + i * R + 4 * cq);
                d.x = fmaf(x4.x, y4.x, d.x);
                d.y = fmaf(x4.y, y4.y, d.y);
                d.z = fmaf(x4.z, y4.z, d.z);
                d.w = fmaf(x4.w, y4.w, d.w);
            }
            dacc[0] += d.x;
            dacc[1] += d.y;
            dacc[2] += d.z;
            dacc[3] += d.w;
        }
        __syncthreads();  // tile k consumed: its slot may be refilled
    }
    // the 8 warps' tile sums in shared memory (fixed order), then the
    // un-permuted, mirrored Gram and the dots into this block's partial
    double *red = reinterpret_cast<double *>(cpd_smem);  // [R][R]
    double *dred = red + R * R;                           // [nrl][R]
    for (int w = 0; w < 8; ++w) {
        if (warp == w) {
#pragma unroll
            for (int q = 0; q < kTiles; ++q) {
                const int mb = q < 4 ? 0 : 1, nb = q < 4 ? q : q - 2;
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int m = mb * 16 + g + ((e & 2) ? 8 : 0);  // logical row
                    const int n = nb * 8 + 2 * t + (e & 1);           // logical column
                    const int pm = (m % 8) * 4 + m / 8, pn = (n % 8) * 4 + n / 8;  // physical columns
                    double &slot = red[pm * R + pn];
                    slot = (w == 0 ? 0.0 : slot) + acc[q][e];
                }
            }
        }
        __syncthreads();
    }
    if (rl < nrl) {
#pragma unroll
        for (int c = 0; c < 4; ++c) dred[rl * R + 4 * cq + c] = dacc[c];
    }
    __syncthreads();
    constexpr int W = R * R + R;
    double *out = part + static_cast<int64_t>(blockIdx.x) * W;
    for (int q = tid; q < R * R; q += blockDim.x) {
        const int a = q / R, b = q % R;
        // the computed block triangle: logical (m, n) with m/16 <= n/16, i.e. computed iff
        // (logical index of a) block <= (logical index of b) block; take that entry or its mirror
        const int la = (a % 4) * 8 + a / 4, lb = (b % 4) * 8 + b / 4;  // physical -> logical
        out[q] = (la / 16 <= lb / 16) ? red[q] : red[b * R + a];
    }
    if (tid < R) {
        double d = 0.0;
        for (int l = 0; l < nrl; ++l) d += dred[l * R + tid];
        out[R * R + tid] = d;
    }
}

// The one dense pass of an iteration at R = 32 (tensor cores, 3xTF32): every
// 128-row tile of M and of the stored factor F arrives once through the
// bulk-copy ring, and per 16-row slab of the tile the warps
//   (1) accumulate the Gram M^T M (gram_tc32_kernel's permuted-column MMAs),
//   (2) accumulate the column dots M o F (the fit's <X, Xhat>; F is the
//       factor the MTTKRP read),
//   (3) compute F_new = M W with K permuted so that thread (g, t) reads
//       physical columns 8t..8t+7 of its two rows (two LDS.128 each):
//       logical k = 8 ks + kk maps to physical column 8 (kk % 4) + 2 ks + kk / 4,
//       and W's fragments (loaded once, split hi/lo, in registers) use the
//       same map; the result is stored over the same rows of F (unless a fit-only iteration:
//       store == 0, or *skip set by the device loop).
// Warp roles: warps [0, W) do (1)-(2) and warps [W, 2W) do (3) on the same
// 16-row slabs, each warp taking slabs rw, rw + W, ... of a tile, so the two
// MMA streams interleave on the tensor pipe (with 8 warps doing all three,
// 240 registers each, the pass ran at 2 warps per scheduler: 102 us on c3,
// tensor pipe 42 % and DRAM 40 % busy; 16 warps in one block per SM: 94 us;
// W = 4 with two 256-thread blocks per SM, each with its own 3-deep ring:
// 88 us).  F's old rows are read by (2) from the ring, and (3) stores the new
// rows straight to global memory: the ring slot is only refilled after the
// tile's barrier.
#ifndef SYSTEC_CPD_PASS_WARPS
#define SYSTEC_CPD_PASS_WARPS 4  // warps per role: 4 = 256-thread blocks, two per SM (c3 pass 88 us);
                                 // 8 = 512 threads, one per SM, 5-deep ring (94 us)
#endif
#ifndef SYSTEC_CPD_PASS_RING
#define SYSTEC_CPD_PASS_RING (SYSTEC_CPD_PASS_WARPS == 8 ? 5 : 3)
#endif
constexpr int kPassRing = SYSTEC_CPD_PASS_RING;
constexpr int kRoleWarps = SYSTEC_CPD_PASS_WARPS;
constexpr int kPassThreads = 64 * kRoleWarps;
constexpr int kPassBlocksPerSm = 8 / kRoleWarps;
static_assert(kRoleWarps == 4 || kRoleWarps == 8, "warps per role: 4 or 8");
static_assert(kPassBlocksPerSm <= SYSTEC_CPD_BPS, "the partial-sum scratch holds SYSTEC_CPD_BPS blocks per SM");
#ifdef SYSTEC_EXP_PASS_EMPTY  // experiment builds only: the ring alone (no MMAs, dots or stores)
constexpr bool kPassCompute = false;
#else
constexpr bool kPassCompute = true;
#endif
__global__ void __launch_bounds__(kPassThreads, kPassBlocksPerSm) pass_tc32_kernel(const float *__restrict__ M, float *F,
                                                                    const float *__restrict__ W, int64_t dim,
                                                                    double *__restrict__ part, int store,
                                                                    const int *skip) {
    constexpr int R = 32;
    extern __shared__ __align__(16) unsigned char cpd_smem[];
    const bool write = store && !(skip && *skip);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
    const bool gram_role = warp < kRoleWarps;
    const int rw = warp % kRoleWarps;  // the warp's slabs: rows 16 (rw + kRoleWarps i) of each 128-row tile
    const int64_t rows = (dim + gridDim.x - 1) / gridDim.x;
    const int64_t lo = blockIdx.x * rows, hi = min(dim, lo + rows);
    TileRingT<kPassRing> tr{reinterpret_cast<float *>(cpd_smem),
                            reinterpret_cast<uint64_t *>(cpd_smem + ring_bytes<kPassRing>(2, R) - kPassRing * 8),
                            M, F, 2, R, lo, hi};
    const int64_t nt = lo < hi ? tr.ntiles() : 0;
    if (tid == 0) {
        tr.init();
        for (int64_t q = 0; q < min(static_cast<int64_t>(kPassRing - 1), nt); ++q) tr.issue(q);
    }
    __syncthreads();
    constexpr int kTiles = 6;  // Gram output tiles (mb, nb): (0,0) (0,1) (0,2) (0,3) (1,2) (1,3)
    double *red = reinterpret_cast<double *>(cpd_smem);  // [R][R] after the loop
    double *dred = red + R * R;                           // [8 warps][4 row lanes][R]
    if (gram_role) {
        double acc[kTiles][4];
#pragma unroll
        for (int q = 0; q < kTiles; ++q)
#pragma unroll
            for (int e = 0; e < 4; ++e) acc[q][e] = 0.0;
        double dacc[4] = {0.0, 0.0, 0.0, 0.0};
        const int dr = lane >> 3, dq = lane & 7;  // column dots: row dr + 4j of the slab, float4 column dq
        for (int64_t k = 0; k < nt; ++k) {
            const int nr = static_cast<int>(min(static_cast<int64_t>(kTileRows), hi - lo - k * kTileRows));
            if (tid == 0 && k + kPassRing - 1 < nt) {
                fence_proxy_async_smem();
                tr.issue(k + kPassRing - 1);
            }
            const float *tx = tr.tile(k, 0), *ty = tr.tile(k, 1);
            tr.wait(k);
#pragma unroll 1
            for (int sl = 0; sl < 8 / kRoleWarps; ++sl) {
            const int w0 = (rw + kRoleWarps * sl) * 16;
            if (kPassCompute && w0 < nr) {
                // (1) Gram
                float f[kTiles][4];
#pragma unroll
                for (int q = 0; q < kTiles; ++q)
#pragma unroll
                    for (int e = 0; e < 4; ++e) f[q][e] = 0.f;
#pragma unroll
                for (int ks = 0; ks < 2; ++ks) {
                    const int q0 = w0 + ks * 8 + t, q1 = q0 + 4;  // rows past nr are zero-weighted
                    const float4 v0 = q0 < nr ? *reinterpret_cast<const float4 *>(tx + q0 * R + 4 * g) : make_float4(0.f, 0.f, 0.f, 0.f);
                    const float4 v1 = q1 < nr ? *reinterpret_cast<const float4 *>(tx + q1 * R + 4 * g) : make_float4(0.f, 0.f, 0.f, 0.f);
                    uint32_t bh[4][2], bl[4][2];
                    split_tf32(v0.x, bh[0][0], bl[0][0]); split_tf32(v1.x, bh[0][1], bl[0][1]);
                    split_tf32(v0.y, bh[1][0], bl[1][0]); split_tf32(v1.y, bh[1][1], bl[1][1]);
                    split_tf32(v0.z, bh[2][0], bl[2][0]); split_tf32(v1.z, bh[2][1], bl[2][1]);
                    split_tf32(v0.w, bh[3][0], bl[3][0]); split_tf32(v1.w, bh[3][1], bl[3][1]);
#pragma unroll
                    for (int mb = 0; mb < 2; ++mb) {
                        const uint32_t ah[4] = {bh[2 * mb][0], bh[2 * mb + 1][0], bh[2 * mb][1], bh[2 * mb + 1][1]};
                        const uint32_t al[4] = {bl[2 * mb][0], bl[2 * mb + 1][0], bl[2 * mb][1], bl[2 * mb + 1][1]};
#pragma unroll
                        for (int nb = 2 * mb; nb < 4; ++nb) {
                            const int q = mb == 0 ? nb : 2 + nb;
                            mma3(f[q], ah, al, bh[nb][0], bh[nb][1], bl[nb][0], bl[nb][1]);
                        }
                    }
                }
#pragma unroll
                for (int q = 0; q < kTiles; ++q)
#pragma unroll
                    for (int e = 0; e < 4; ++e) acc[q][e] += f[q][e];
                // (2) column dots M o F over the slab's rows
                float4 d = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int i = w0 + dr + 4 * j;
                    if (i < nr) {
                        const float4 x4 = *reinterpret_cast<const float4 *>(tx + i * R + 4 * dq);
                        const float4 y4 = *reinterpret_cast<const float4 *>(ty + i * R + 4 * dq);
                        d.x = fmaf(x4.x, y4.x, d.x);
                        d.y = fmaf(x4.y, y4.y, d.y);
                        d.z = fmaf(x4.z, y4.z, d.z);
                        d.w = fmaf(x4.w, y4.w, d.w);
                    }
                }
                dacc[0] += d.x;
                dacc[1] += d.y;
                dacc[2] += d.z;
                dacc[3] += d.w;
            }
            }
            __syncthreads();  // tile k consumed by every warp: its slot may be refilled
        }
        // the 8 gram warps' sums in shared memory in a fixed order (named
        // barrier 1: these warps only; the ring is idle once every tile's
        // block barrier has passed), un-permuted below
        for (int w = 0; w < kRoleWarps; ++w) {
            if (warp == w) {
#pragma unroll
                for (int q = 0; q < kTiles; ++q) {
                    const int mb = q < 4 ? 0 : 1, nb = q < 4 ? q : q - 2;
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const int m = mb * 16 + g + ((e & 2) ? 8 : 0);
                        const int n = nb * 8 + 2 * t + (e & 1);
                        const int pm = (m % 8) * 4 + m / 8, pn = (n % 8) * 4 + n / 8;
                        double &slot = red[pm * R + pn];
                        slot = (w == 0 ? 0.0 : slot) + acc[q][e];
                    }
                }
            }
            asm volatile("bar.sync 1, %0;" ::"n"(32 * kRoleWarps) : "memory");
        }
#pragma unroll
        for (int c = 0; c < 4; ++c) dred[(warp * 4 + dr) * R + 4 * dq + c] = dacc[c];
    } else {
        uint32_t wh[4][4][2], wl[4][4][2];  // W fragments, permuted K
#pragma unroll
        for (int ks = 0; ks < 4; ++ks)
#pragma unroll
            for (int nb = 0; nb < 4; ++nb) {
                const int k0 = 8 * t + 2 * ks, k1 = k0 + 1;
                split_tf32(W[k0 * R + nb * 8 + g], wh[ks][nb][0], wl[ks][nb][0]);
                split_tf32(W[k1 * R + nb * 8 + g], wh[ks][nb][1], wl[ks][nb][1]);
            }
        for (int64_t k = 0; k < nt; ++k) {
            const int64_t r0g = lo + k * kTileRows;
            const int nr = static_cast<int>(min(static_cast<int64_t>(kTileRows), hi - r0g));
            const float *tx = tr.tile(k, 0);
            tr.wait(k);
#pragma unroll 1
            for (int sl = 0; sl < 8 / kRoleWarps; ++sl) {
            const int w0 = (rw + kRoleWarps * sl) * 16;
            if (kPassCompute && write && w0 < nr) {
                // (3) F_new = M W for the slab
                const int ra = w0 + g, rb = ra + 8;  // rows past nr: computed, never stored
                float o[4][4];
#pragma unroll
                for (int nb = 0; nb < 4; ++nb)
#pragma unroll
                    for (int e = 0; e < 4; ++e) o[nb][e] = 0.f;
                const float4 a0 = *reinterpret_cast<const float4 *>(tx + ra * R + 8 * t);
                const float4 a1 = *reinterpret_cast<const float4 *>(tx + ra * R + 8 * t + 4);
                const float4 b0 = *reinterpret_cast<const float4 *>(tx + rb * R + 8 * t);
                const float4 b1 = *reinterpret_cast<const float4 *>(tx + rb * R + 8 * t + 4);
                const float ra8[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
                const float rb8[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
                for (int ks = 0; ks < 4; ++ks) {
                    uint32_t ah[4], al[4];
                    split_tf32(ra8[2 * ks], ah[0], al[0]);
                    split_tf32(rb8[2 * ks], ah[1], al[1]);
                    split_tf32(ra8[2 * ks + 1], ah[2], al[2]);
                    split_tf32(rb8[2 * ks + 1], ah[3], al[3]);
#pragma unroll
                    for (int nb = 0; nb < 4; ++nb)
                        mma3(o[nb], ah, al, wh[ks][nb][0], wh[ks][nb][1], wl[ks][nb][0], wl[ks][nb][1]);
                }
                float *fa = F + (r0g + ra) * R + 2 * t, *fb = F + (r0g + rb) * R + 2 * t;
#pragma unroll
                for (int nb = 0; nb < 4; ++nb) {
                    if (ra < nr) *reinterpret_cast<float2 *>(fa + nb * 8) = make_float2(o[nb][0], o[nb][1]);
                    if (rb < nr) *reinterpret_cast<float2 *>(fb + nb * 8) = make_float2(o[nb][2], o[nb][3]);
                }
            }
            }
            __syncthreads();  // tile k consumed by every warp: its slot may be refilled
        }
    }
    __syncthreads();  // the ring is idle: its memory holds the reductions
    constexpr int Wd = R * R + R;
    double *out = part + static_cast<int64_t>(blockIdx.x) * Wd;
    for (int q = tid; q < R * R; q += blockDim.x) {
        const int a = q / R, b = q % R;
        const int la = (a % 4) * 8 + a / 4, lb = (b % 4) * 8 + b / 4;
        out[q] = (la / 16 <= lb / 16) ? red[q] : red[b * R + a];
    }
    if (tid < R) {
        double d = 0.0;
        for (int l = 0; l < 4 * kRoleWarps; ++l) d += dred[l * R + tid];
        out[R * R + tid] = d;
    }
}

// The same partial sums for R % 4 == 0, R <= 32 (aligned rows): tiles arrive
// through the bulk-copy ring, and only the upper triangle of 4x4 micro-tiles
// (a-block <= b-block: 36 of 64 at R = 32) is accumulated and mirrored at the
// end — the Gram matrix is symmetric.  Row pointers advance by increments (no
// per-row index arithmetic); the column dots use float4 lanes.  Per row at
// R = 32: 36 threads x (2 LDS.128 + 16 FFMA) instead of 64.
__global__ void __launch_bounds__(256) gram_dots_sym_kernel(const float *__restrict__ B, const float *__restrict__ M,
                                                            int64_t dim, int R, double *__restrict__ part) {
    extern __shared__ __align__(16) unsigned char cpd_smem[];
    const int T4 = R / 4;
    const int NT = T4 * (T4 + 1) / 2;  // upper-triangle micro-tiles
    const int RG = blockDim.x / NT;    // row groups
    const int tid = threadIdx.x;
    const int mt = tid % NT, g = tid / NT;
    const bool active = g < RG;
    int a4 = 0, rem = mt;  // mt -> (a4, b4), a4 <= b4, row-major over the upper triangle
    while (rem >= T4 - a4) {
        rem -= T4 - a4;
        ++a4;
    }
    const int b4 = a4 + rem;
    const int cq = tid % T4, rl = tid / T4, nrl = blockDim.x / T4;  // column dots: (row lane, float4 column)
    const int64_t rows = (dim + gridDim.x - 1) / gridDim.x;
    const int64_t lo = blockIdx.x * rows, hi = min(dim, lo + rows);
    TileRing tr{reinterpret_cast<float *>(cpd_smem), reinterpret_cast<uint64_t *>(cpd_smem + ring_bytes(2, R) - kRingS * 8),
                B, M, 2, R, lo, hi};
    const int64_t nt = lo < hi ? tr.ntiles() : 0;
    if (tid == 0) {
        tr.init();
        for (int64_t q = 0; q < min(static_cast<int64_t>(kRingS - 1), nt); ++q) tr.issue(q);
    }
    __syncthreads();
    double acc[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) acc[k] = 0.0;
    double dacc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int64_t k = 0; k < nt; ++k) {
        const int nr = static_cast<int>(min(static_cast<int64_t>(kTileRows), hi - lo - k * kTileRows));
        if (tid == 0 && k + kRingS - 1 < nt) {
            fence_proxy_async_smem();
            tr.issue(k + kRingS - 1);
        }
        const float *tb = tr.tile(k, 0), *tm = tr.tile(k, 1);
        tr.wait(k);
        if (active && g < nr) {
            float f[16];
#pragma unroll
            for (int q = 0; q < 16; ++q) f[q] = 0.f;
            const float *px = tb + g * R + 4 * a4, *py = tb + g * R + 4 * b4;
            const float *pend = tb + nr * R;
            const int step = RG * R;
#pragma unroll 2
            for (; px < pend; px += step, py += step) {
                const float4 x = *reinterpret_cast<const float4 *>(px);
                const float4 y = *reinterpret_cast<const float4 *>(py);
                const float xa[4] = {x.x, x.y, x.z, x.w}, yb[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
                for (int u = 0; u < 4; ++u)
#pragma unroll
                    for (int v = 0; v < 4; ++v) f[u * 4 + v] = fmaf(xa[u], yb[v], f[u * 4 + v]);
            }
#pragma unroll
            for (int q = 0; q < 16; ++q) acc[q] += f[q];
        }
        if (rl < nrl) {
            float4 d = make_float4(0.f, 0.f, 0.f, 0.f);
            for (int i = rl; i < nr; i += nrl) {
                const float4 m4 = *reinterpret_cast<const float4 *>(tm + i * R + 4 * cq);
                const float4 b4v = *reinterpret_cast<const float4 *>(tb + i * R + 4 * cq);
                d.x = fmaf(m4.x, b4v.x, d.x);
                d.y = fmaf(m4.y, b4v.y, d.y);
                d.z = fmaf(m4.z, b4v.z, d.z);
                d.w = fmaf(m4.w, b4v.w, d.w);
            }
            dacc[0] += d.x;
            dacc[1] += d.y;
            dacc[2] += d.z;
            dacc[3] += d.w;
        }
        __syncthreads();  // tile k consumed: its slot may be refilled
    }
    // sum the row groups (and the dot lanes) in shared memory; the ring is idle
    double *red = reinterpret_cast<double *>(cpd_smem);  // [NT][16]
    double *dred = red + 36 * 16;                          // [nrl][R]
    for (int grp = 0; grp < RG; ++grp) {
        if (active && g == grp) {
#pragma unroll
            for (int q = 0; q < 16; ++q) red[mt * 16 + q] = (grp == 0 ? 0.0 : red[mt * 16 + q]) + acc[q];
        }
        __syncthreads();
    }
    if (rl < nrl) {
#pragma unroll
        for (int c = 0; c < 4; ++c) dred[rl * R + 4 * cq + c] = dacc[c];
    }
    __syncthreads();
    const int W = R * R + R;
    double *out = part + static_cast<int64_t>(blockIdx.x) * W;
    for (int q = tid; q < NT * 16; q += blockDim.x) {
        const int m = q / 16, e = q % 16;
        int ta = 0, rr = m;
        while (rr >= T4 - ta) {
            rr -= T4 - ta;
            ++ta;
        }
        const int a = ta * 4 + e / 4, b = (ta + rr) * 4 + e % 4;
        out[a * R + b] = red[q];
        out[b * R + a] = red[q];  // mirror (the diagonal tiles write their own mirror image)
    }
    if (tid < R) {
        double d = 0.0;
        for (int l = 0; l < nrl; ++l) d += dred[l * R + tid];
        out[R * R + tid] = d;
    }
}

// R <= 16: the same partial sums with no staging and no barriers in the row
// loop.  Each warp walks its own rows (coalesced 4R-byte loads, 4 rows in
// flight); lane b holds column b of the row and accumulates the whole column
// b of the Gram matrix, acc[a] += x_a x_b with x_a broadcast by a shuffle
// (R shuffles + R FMAs per row), fp32 over <= 32 rows then fp64; lane b also
// accumulates the column dot M[i][b] B[i][b].  The block's 8 warps are summed
// in shared memory (fixed order) into one partial per block.
template <int RT>
__global__ void __launch_bounds__(256) gram_dots_warp_kernel(const float *__restrict__ B, const float *__restrict__ M,
                                                             int64_t dim, int R, double *__restrict__ part) {
    __shared__ double wsum[RT * RT + RT];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t rows = (dim + gridDim.x - 1) / gridDim.x;
    const int64_t lo = blockIdx.x * rows, hi = min(dim, lo + rows);
    const bool col = lane < R;
    double acc[RT];
    double dacc = 0.0;
#pragma unroll
    for (int a = 0; a < RT; ++a) acc[a] = 0.0;
    int64_t i = lo + warp;
    while (i < hi) {
        float f[RT];
#pragma unroll
        for (int a = 0; a < RT; ++a) f[a] = 0.f;
        float d = 0.f;
        // up to 32 rows per fp32 block, 4 loaded ahead
#pragma unroll 1
        for (int blk = 0; blk < 8 && i < hi; ++blk) {
            float x[4], m[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int64_t r = i + static_cast<int64_t>(u) * 8;
                const bool ok = col && r < hi;
                x[u] = ok ? __ldg(B + r * R + lane) : 0.f;
                m[u] = ok ? __ldg(M + r * R + lane) : 0.f;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                d = fmaf(m[u], x[u], d);
#pragma unroll
                for (int a = 0; a < RT; ++a) f[a] = fmaf(__shfl_sync(0xffffffffu, x[u], a), x[u], f[a]);
            }
            i += 32;
        }
#pragma unroll
        for (int a = 0; a < RT; ++a) acc[a] += f[a];
        dacc += d;
    }
    // warp partials summed into shared memory one warp at a time (fixed order);
    // column b of the Gram matrix is lane b's acc[]
    for (int w = 0; w < (blockDim.x >> 5); ++w) {
        if (warp == w && col) {
#pragma unroll
            for (int a = 0; a < RT; ++a)
                if (a < R) wsum[a * R + lane] = (w == 0 ? 0.0 : wsum[a * R + lane]) + acc[a];
            wsum[R * R + lane] = (w == 0 ? 0.0 : wsum[R * R + lane]) + dacc;
        }
        __syncthreads();
    }
    const int W = R * R + R;
    for (int q = threadIdx.x; q < W; q += blockDim.x) part[static_cast<int64_t>(blockIdx.x) * W + q] = wsum[q];
}

// out[q] = sum_blk part[blk][q], q < width: one warp per output, lanes stride
// over the blocks, shuffle-reduced (fixed order: deterministic)
__global__ void reduce_partials_kernel(const double *__restrict__ part, int blocks, int width,
                                       double *__restrict__ out, const int *skip) {
    if (skip && *skip) return;
    const int q = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (q >= width) return;
    double s = 0.0;
    for (int b = lane; b < blocks; b += 32) s += part[static_cast<int64_t>(b) * width + q];
#pragma unroll
    for (int d = 16; d; d >>= 1) s += __shfl_down_sync(0xffffffffu, s, d);
    if (lane == 0) out[q] = s;
}

// ||X||^2 = sum_e v_e^2 orbit_e over the plan's canonical stream
template <int N>
__global__ void tensor_norm_kernel(const int32_t *__restrict__ coords, int64_t ld, const float *__restrict__ vals,
                                   int64_t nnz, double *__restrict__ out) {
    double acc = 0.0;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x) {
        int run = 1;
        double denom = 1.0, f = 1.0;
        int32_t prev = coords[e];
        for (int t = 1; t < N; ++t) {
            const int32_t c = coords[t * ld + e];
            if (c == prev) {
                ++run;
                f *= run;
            } else {
                denom *= f;
                run = 1;
                f = 1.0;
            }
            prev = c;
        }
        denom *= f;
        double nf = 1.0;
        for (int k = 2; k <= N; ++k) nf *= k;
        const double v = vals[e];
        acc += v * v * (nf / denom);
    }
    for (int d = 16; d; d >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, d);
    if ((threadIdx.x & 31) == 0) atomicAdd(out, acc);
}

// The R x R algebra of an iteration, one block of 1024 threads, fp64.
//
// State (fp64, per column r): lambda_r of the current iterate B (unit
// columns), the scale t_r of the stored factor F = B diag(t), and the divisor
// lt_r folded into W when it was built.  G_B = B^T B is carried.  The MTTKRP
// reads F, so M = MTTKRP(X, F) = MTTKRP(X, B) diag(t)^{n-1} (multilinearity).
//   FIT      <X, Xhat> = sum_r lambda_r dots_r / t_r^n  (dots = sum_i M o F),
//            ||Xhat||^2 = lambda^T G_B^{.n} lambda.
//   UPDATE   the pass writes F_new = M W = B_new diag(lambda_new / lt), so
//            P = F_new^T F_new = W^T G_M W,  t = sqrt(diag P),
//            lambda = t lt,  G_B = diag(1/t) P diag(1/t).
//   PRENORM  (two-pass form, iteration 0, before the pass writes)
//            W <- W diag(1/t), t = 1: the pass then writes the unit-column
//            B_new itself.  lambda_1 carries the caller's column norms c of
//            B_0 (lambda_1 ~ c^{-(n-1)}), so the next prediction is taken
//            as pf lambda with pf = c^{n-1} (a unit-column B_0's lambda_1).
//   SOLVE    H = G_B^{.(n-1)}, equilibrated to unit diagonal with a 1e-12
//            ridge, H^{-1} by in-place Gauss-Jordan elimination (SPD: no
//            pivoting), and the next
//            pass's W = diag(t)^{-(n-1)} H^{-1} diag(1/lt) with lt = pf lambda
//            (pf = 1 after iteration 0): B_new = MTTKRP(X, B) H^{-1}
//            diag(1/lambda_new) and the current lambda predicts lambda_new,
//            so the stored F stays near unit columns (t = lambda_new /
//            lambda) without a pass of its own.
// A zero column (lambda = 0) keeps t = lt = 1.  UPDATE, PRENORM and SOLVE
// are dropped when *skip (the device loop's fit-only iteration).  H lives in
// registers: thread t owns row t / TPR and the CW columns [k*CW, (k+1)*CW),
// k = t % TPR (TPR = 16, 32, 16 for R <= 16, 32, 48; CW = 1, 1, 3); each
// elimination step publishes the pivot row, column and reciprocal through
// shared memory (double-buffered: one barrier per step).
enum : int { kFit = 1, kUpdate = 2, kSolve = 4, kPrenorm = 8 };
struct CpdCols {
    double *lam, *t, *lt, *pf;  // [R] each
};
// threads of the small block: the inverse's pivot steps run fastest with one
// column per thread (460 cycles per step at R = 32, against 1,150 with 256
// threads, 4 columns each, and 1,230 on one warp holding the rows in
// registers with shuffled pivots; clock64 phases,
// profiles/r02/cpd_small_phase_clocks.log)
constexpr int kSmallThreads = 1024;
constexpr int pow2_floor(int x) { return x >= 2 ? 2 * pow2_floor(x / 2) : 1; }
template <int RC>  // rank class: R <= RC (16, 32, 48)
__global__ void __launch_bounds__(kSmallThreads, 1) cp_small_kernel(double *__restrict__ GB, int R, int n,
                                                                    CpdCols cols, const double *__restrict__ dots,
                                                                    double *__restrict__ xhat2,
                                                                    const double *__restrict__ GM,
                                                                    float *__restrict__ W, int flags, const int *skip) {
    // H: thread t owns row t / TPR and the CW columns [k*CW, (k+1)*CW), k = t % TPR
    constexpr int kT = kSmallThreads;
    constexpr int TPR = pow2_floor(kT / RC) < RC ? pow2_floor(kT / RC) : RC;
    constexpr int CW = (RC + TPR - 1) / TPR;
    constexpr int kPq = (kMaxCpR * kMaxCpR + kT - 1) / kT;
    // every operand is staged in shared memory first (one coalesced load each):
    // the block is a single SM, and dependent global loads were most of its time
    extern __shared__ __align__(16) unsigned char cpd_smem[];
    const int RR = R * R;
    double *As = reinterpret_cast<double *>(cpd_smem);  // W
    double *Gs = As + RR;                                // G_M
    double *Ts = Gs + RR;                                // G_M W, then P, then G_B
    double *Bs = Ts + RR;                                // G_B (current)
    double *lam = Bs + RR, *ts = lam + R, *lt = ts + R, *pf = lt + R, *dt = pf + R, *eq = dt + R;
    __shared__ double piv[2][2 * kMaxCpR];
    __shared__ double fcol[2][kMaxCpR];
    __shared__ double pinv[2];
    __shared__ double red[32];
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, wid = tid >> 5;
    const bool skipped = skip && *skip;
    const bool fit = flags & kFit, update = (flags & kUpdate) && !skipped, solve = (flags & kSolve) && !skipped;
    const bool prenorm = (flags & kPrenorm) && !skipped;
#ifdef SYSTEC_EXP_SMALL_CLOCKS  // experiment builds: phase timestamps of the small block
    long long clk[8];
    clk[0] = clock64();
#define SMALL_CLK(i) (clk[i] = clock64())
#else
#define SMALL_CLK(i) ((void)0)
#endif
    for (int q = tid; q < RR; q += nt) {
        Bs[q] = GB[q];
        if (update) {
            As[q] = W[q];
            Gs[q] = GM[q];
        }
    }
    if (tid < R) {
        lam[tid] = cols.lam[tid];
        ts[tid] = cols.t[tid];
        lt[tid] = cols.lt[tid];
        pf[tid] = cols.pf[tid];
        dt[tid] = dots[tid];
    }
    __syncthreads();
    SMALL_CLK(1);
    if (fit) {  // of the current iterate: before G_B, lambda, t change
        double part = 0.0;
        for (int q = tid; q < RR; q += nt) {
            const int a = q / R, b = q % R;
            const double gp = Bs[q];
            double h = 1.0;
            for (int e = 0; e < n; ++e) h *= gp;
            part += lam[a] * lam[b] * h;
        }
#pragma unroll
        for (int d = 16; d; d >>= 1) part += __shfl_down_sync(0xffffffffu, part, d);
        if (lane == 0) red[wid] = part;
        __syncthreads();
        if (tid < 32) {
            double v = tid < nt / 32 ? red[tid] : 0.0;
            double ip = 0.0;
            for (int a = tid; a < R; a += 32) {
                double tn = 1.0;
                for (int e = 0; e < n; ++e) tn *= ts[a];
                ip += lam[a] * dt[a] / tn;
            }
#pragma unroll
            for (int d = 16; d; d >>= 1) {
                v += __shfl_down_sync(0xffffffffu, v, d);
                ip += __shfl_down_sync(0xffffffffu, ip, d);
            }
            if (tid == 0) {
                xhat2[0] = v;
                xhat2[1] = ip;
            }
        }
    }
    SMALL_CLK(2);
    if (!update && !solve) return;  // block-uniform
    __syncthreads();
    if constexpr (RC <= 32) {
        if (update) {
            // T = G_M W, then P = W^T T: warp w < 8 owns rows w, w + 8, w + 16,
            // w + 24, lane b the column; each W (or T) element read serves four
            // rows (6.8k against 10k cycles for one output per thread of 1024)
            const int b = wid < 8 ? lane : R;
            double acc[4] = {0.0, 0.0, 0.0, 0.0};
            if (b < R)
                for (int c = 0; c < R; ++c) {
                    const double wcb = As[c * R + b];
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const int a = wid + 8 * i;
                        if (a < R) acc[i] = fma(Gs[a * R + c], wcb, acc[i]);
                    }
                }
#pragma unroll
            for (int i = 0; i < 4; ++i)
                if (wid + 8 * i < R && b < R) Ts[(wid + 8 * i) * R + b] = acc[i];
            __syncthreads();
#pragma unroll
            for (int i = 0; i < 4; ++i) acc[i] = 0.0;
            if (b < R)
                for (int c = 0; c < R; ++c) {
                    const double tcb = Ts[c * R + b];
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const int a = wid + 8 * i;
                        if (a < R) acc[i] = fma(As[c * R + a], tcb, acc[i]);
                    }
                }
            __syncthreads();
#pragma unroll
            for (int i = 0; i < 4; ++i)
                if (wid + 8 * i < R && b < R) Ts[(wid + 8 * i) * R + b] = acc[i];
            __syncthreads();
        }
    } else if (update) {
        // four independent partial sums per output (short dependent DFMA chains otherwise)
        for (int q = tid; q < RR; q += nt) {  // T = G_M W
            const int a = q / R, b = q % R;
            const double *g = Gs + a * R;
            double t0 = 0.0, t1 = 0.0, t2 = 0.0, t3 = 0.0;
            int c = 0;
            for (; c + 4 <= R; c += 4) {
                t0 = fma(g[c], As[c * R + b], t0);
                t1 = fma(g[c + 1], As[(c + 1) * R + b], t1);
                t2 = fma(g[c + 2], As[(c + 2) * R + b], t2);
                t3 = fma(g[c + 3], As[(c + 3) * R + b], t3);
            }
            for (; c < R; ++c) t0 = fma(g[c], As[c * R + b], t0);
            Ts[q] = (t0 + t1) + (t2 + t3);
        }
        __syncthreads();
        double Pq[kPq];  // P = W^T T
#pragma unroll
        for (int u = 0; u < kPq; ++u) {
            Pq[u] = 0.0;
            const int q = tid + u * nt;
            if (q < RR) {
                const int a = q / R, b = q % R;
                double t0 = 0.0, t1 = 0.0, t2 = 0.0, t3 = 0.0;
                int c = 0;
                for (; c + 4 <= R; c += 4) {
                    t0 = fma(As[c * R + a], Ts[c * R + b], t0);
                    t1 = fma(As[(c + 1) * R + a], Ts[(c + 1) * R + b], t1);
                    t2 = fma(As[(c + 2) * R + a], Ts[(c + 2) * R + b], t2);
                    t3 = fma(As[(c + 3) * R + a], Ts[(c + 3) * R + b], t3);
                }
                for (; c < R; ++c) t0 = fma(As[c * R + a], Ts[c * R + b], t0);
                Pq[u] = (t0 + t1) + (t2 + t3);
            }
        }
        __syncthreads();
#pragma unroll
        for (int u = 0; u < kPq; ++u)
            if (tid + u * nt < RR) Ts[tid + u * nt] = Pq[u];
        __syncthreads();
    }
    if (update) {  // Ts = P = F_new^T F_new
        if (tid < R) {
            const double d = Ts[tid * R + tid];
            const double tn = sqrt(d > 0.0 ? d : 0.0);
            lam[tid] = tn * lt[tid];
            ts[tid] = tn > 0.0 ? tn : 1.0;
            if (prenorm) {  // G_B still holds B_0's Gram: pf = c^{n-1}
                const double c2 = Bs[tid * R + tid];
                pf[tid] = c2 > 0.0 ? pow(c2, 0.5 * (n - 1)) : 1.0;
            }
        }
        __syncthreads();
        for (int q = tid; q < RR; q += nt) {
            const int a = q / R, b = q % R;
            const double g = Ts[q] / (ts[a] * ts[b]);
            Ts[q] = g;
            GB[q] = g;
            if (prenorm) W[q] = static_cast<float>(As[q] / ts[b]);
        }
        __syncthreads();
        if (prenorm && tid < R) ts[tid] = 1.0;
    } else {
        for (int q = tid; q < RR; q += nt) Ts[q] = Bs[q];
    }
    SMALL_CLK(3);
    if (solve) {
        __syncthreads();
        // H = G_B^{.(n-1)}, equilibrated to unit diagonal (eq = diag(H)^{-1/2};
        // the caller's factor may scale its columns arbitrarily) with a 1e-12
        // ridge, inverted in place by Gauss-Jordan elimination:
        // H^{-1} = diag(eq) (diag(eq) H diag(eq) + 1e-12 I)^{-1} diag(eq)
        if (tid < R) {
            double h = 1.0;
            for (int q = 0; q < n - 1; ++q) h *= Ts[tid * R + tid];
            eq[tid] = h > 0.0 ? 1.0 / sqrt(h) : 1.0;
        }
        __syncthreads();
        const int row = tid / TPR, k = tid % TPR;
        const bool own = row < R;
        const int c0 = k * CW;
        double A[CW];
#pragma unroll
        for (int u = 0; u < CW; ++u) {
            const int c = c0 + u;
            double v = 0.0;
            if (own && c < R) {
                const double gp = Ts[row * R + c];
                double h = 1.0;
                for (int q = 0; q < n - 1; ++q) h *= gp;
                v = h * eq[row] * eq[c] + (c == row ? 1e-12 : 0.0);
            }
            A[u] = v;
        }
        SMALL_CLK(4);
        // in place: after step j, column j holds the inverse's column; the
        // pivot row / column / reciprocal are double-buffered in shared
        // memory, so one barrier per step suffices (a thread can only
        // overwrite a buffer after every thread passed the next step's barrier)
        for (int j = 0; j < R; ++j) {
            const int bsel = j & 1;
#pragma unroll
            for (int u = 0; u < CW; ++u) {
                const int c = c0 + u;
                if (own && c < R) {
                    if (c == j) fcol[bsel][row] = A[u];
                    if (row == j) piv[bsel][c] = A[u];
                    if (row == j && c == j) pinv[bsel] = 1.0 / A[u];  // one division per step
                }
            }
            __syncthreads();
            if (own) {
                const double pv = pinv[bsel];
                const double f = fcol[bsel][row] * pv;
#pragma unroll
                for (int u = 0; u < CW; ++u) {
                    const int c = c0 + u;
                    if (c < R) {
                        if (row == j) A[u] = (c == j) ? pv : A[u] * pv;
                        else A[u] = (c == j) ? -f : fma(-f, piv[bsel][c], A[u]);
                    }
                }
            }
        }
        SMALL_CLK(5);
        // W = diag(t)^{-(n-1)} H^{-1} diag(1/lt), lt = pf lambda
#pragma unroll
        for (int u = 0; u < CW; ++u) {
            const int c = c0 + u;
            if (own && c < R) {
                double tp = 1.0;
                for (int q = 0; q < n - 1; ++q) tp *= ts[row];
                const double lb = lam[c] > 0.0 ? lam[c] * pf[c] : 1.0;
                W[row * R + c] = static_cast<float>(A[u] * eq[row] * eq[c] / (tp * lb));
            }
        }
    }
    __syncthreads();
#ifdef SYSTEC_EXP_SMALL_CLOCKS
    if (tid == 0) {
        SMALL_CLK(6);
        printf("small flags=%d R=%d cycles: stage %lld fit %lld upd %lld build %lld gj %lld w %lld\n", flags, R,
               clk[1] - clk[0], clk[2] - clk[1], clk[3] - clk[2], clk[4] - clk[3], clk[5] - clk[4], clk[6] - clk[5]);
    }
#endif
    if (tid < R) {
        cols.lam[tid] = lam[tid];
        cols.t[tid] = ts[tid];
        if (solve) {
            cols.lt[tid] = lam[tid] > 0.0 ? lam[tid] * pf[tid] : 1.0;
            cols.pf[tid] = 1.0;
        } else {
            cols.pf[tid] = pf[tid];
        }
    }
}
size_t small_smem_bytes(int R) { return (4ull * R * R + 6ull * R) * sizeof(double); }

// F /= t column-wise (the unit-column factor on return; one float
// reciprocal per column, float4 lanes when R % 4 == 0) and lambda (fp32)
__global__ void cp_finish_kernel(float *__restrict__ F, int64_t dim, int R, CpdCols cols, float *__restrict__ lam) {
    __shared__ float rinv[kMaxCpR];
    if (threadIdx.x < R) rinv[threadIdx.x] = static_cast<float>(1.0 / cols.t[threadIdx.x]);
    __syncthreads();
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    const int64_t first = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (R % 4 == 0 && (reinterpret_cast<uintptr_t>(F) & 15u) == 0) {
        float4 *F4 = reinterpret_cast<float4 *>(F);
        const int R4 = R / 4;
        const int64_t total4 = dim * R4;
        for (int64_t q = first; q < total4; q += stride) {
            const int c = static_cast<int>(q % R4) * 4;
            float4 v = F4[q];
            v.x *= rinv[c];
            v.y *= rinv[c + 1];
            v.z *= rinv[c + 2];
            v.w *= rinv[c + 3];
            F4[q] = v;
        }
    } else {
        for (int64_t q = first; q < dim * R; q += stride) F[q] *= rinv[q % R];
    }
    if (blockIdx.x == 0 && threadIdx.x < R) lam[threadIdx.x] = static_cast<float>(cols.lam[threadIdx.x]);
}

// the caller's factor is the iterate itself: lambda = t = lt = pf = 1
__global__ void cp_cols_init_kernel(CpdCols cols, int R) {
    if (threadIdx.x < R)
        cols.lam[threadIdx.x] = cols.t[threadIdx.x] = cols.lt[threadIdx.x] = cols.pf[threadIdx.x] = 1.0;
}

// Bout = M W (the FFMA form of the pass's F_new = M W; see cp_small_kernel).  RT = R
// rounded up to a multiple of 8: thread (column b, row group) keeps W[:, b] in
// registers and reads each staged M row as 16-byte broadcasts.
template <int RT>
__global__ void __launch_bounds__(256) apply_inverse_kernel(const float *__restrict__ M, const float *__restrict__ Hinv,
                                                            int64_t dim, int R, float *__restrict__ Bout,
                                                            const int *skip, bool ring) {
    if (skip && *skip) return;  // device-side loop: last iteration evaluates the fit only
    // dynamic shared memory: the ring of kRingS tiles of M (bulk copies), or
    // one synchronously staged tile [kTileRows][RT] when the ring cannot run
    extern __shared__ __align__(16) unsigned char cpd_smem[];
    float *Msync = reinterpret_cast<float *>(cpd_smem);
    const int tid = threadIdx.x;
    const int b = tid % RT, rg = tid / RT;
    constexpr int RGN = 256 / RT;
    const bool active = rg < RGN && b < R;
    float h[RT];
#pragma unroll
    for (int a = 0; a < RT; ++a) h[a] = (active && a < R) ? Hinv[a * R + b] : 0.f;
    const int64_t rows = (dim + gridDim.x - 1) / gridDim.x;
    const int64_t lo = blockIdx.x * rows, hi = min(dim, lo + rows);
    TileRing tr{reinterpret_cast<float *>(cpd_smem), reinterpret_cast<uint64_t *>(cpd_smem + ring_bytes(1, R) - kRingS * 8),
                M, nullptr, 1, R, lo, hi};
    const int64_t nt = ring && lo < hi ? tr.ntiles() : 0;
    if (ring) {
        if (tid == 0) {
            tr.init();
            for (int64_t q = 0; q < min(static_cast<int64_t>(kRingS - 1), nt); ++q) tr.issue(q);
        }
        __syncthreads();
    }
    int64_t k = 0;
    for (int64_t r0 = lo; r0 < hi; r0 += kTileRows, ++k) {
        const int nr = static_cast<int>(min(static_cast<int64_t>(kTileRows), hi - r0));
        const float *Ms;
        if (ring) {  // rows of R == RT floats
            if (tid == 0 && k + kRingS - 1 < nt) {
                fence_proxy_async_smem();
                tr.issue(k + kRingS - 1);
            }
            Ms = tr.tile(k, 0);
            tr.wait(k);
        } else {
            stage_rows(Msync, M, r0, nr, R, RT);
            Ms = Msync;
            __syncthreads();
        }
        if (active) {
            // pointer increments (no per-row 64-bit index arithmetic)
            float *o = Bout + (r0 + rg) * R + b;
            const float *mrow = Ms + rg * RT;
            const float *mend = Ms + nr * RT;
            // two rows per step: two independent FMA chains per thread
            for (; mrow + RGN * RT < mend; mrow += 2 * RGN * RT, o += 2 * RGN * R) {
                const float4 *m4 = reinterpret_cast<const float4 *>(mrow);
                const float4 *n4 = reinterpret_cast<const float4 *>(mrow + RGN * RT);
                float s = 0.f, u = 0.f;
#pragma unroll
                for (int a4 = 0; a4 < RT / 4; ++a4) {
                    const float4 x = m4[a4], y = n4[a4];
                    s = fmaf(x.x, h[4 * a4 + 0], s);
                    u = fmaf(y.x, h[4 * a4 + 0], u);
                    s = fmaf(x.y, h[4 * a4 + 1], s);
                    u = fmaf(y.y, h[4 * a4 + 1], u);
                    s = fmaf(x.z, h[4 * a4 + 2], s);
                    u = fmaf(y.z, h[4 * a4 + 2], u);
                    s = fmaf(x.w, h[4 * a4 + 3], s);
                    u = fmaf(y.w, h[4 * a4 + 3], u);
                }
                o[0] = s;
                o[RGN * R] = u;
            }
            for (; mrow < mend; mrow += RGN * RT, o += RGN * R) {
                const float4 *m4 = reinterpret_cast<const float4 *>(mrow);
                float s = 0.f;
#pragma unroll
                for (int a4 = 0; a4 < RT / 4; ++a4) {
                    const float4 x = m4[a4];
                    s = fmaf(x.x, h[4 * a4 + 0], s);
                    s = fmaf(x.y, h[4 * a4 + 1], s);
                    s = fmaf(x.z, h[4 * a4 + 2], s);
                    s = fmaf(x.w, h[4 * a4 + 3], s);
                }
                *o = s;
            }
        }
        __syncthreads();  // tile k consumed: its slot may be refilled
    }
}

// Device-side convergence test of the CP-ALS loop (one thread): the fit of
// the current iterate from the pieces small_solve_kernel wrote, stored in
// fits[it-1]; the loop continues (conditional WHILE node of the iteration
// graph) unless this was the last iteration or |fit - previous| < tol.  The
// body runs MTTKRP -> fit pieces + R x R update -> apply pass -> this test,
// so the skip flag it sets is for the NEXT body run: the last iteration
// evaluates the fit only, as in the host loop.
__global__ void cpd_fit_check_kernel(const double *__restrict__ xhat2, CpdLoopState *st, double *__restrict__ fits,
                                     double tol, int max_iters, cudaGraphConditionalHandle handle) {
    const int it = ++st->it;
    const double x2 = st->x2;
    const double r2 = x2 - 2.0 * xhat2[1] + xhat2[0];
    const double fit = 1.0 - sqrt(r2 > 0.0 ? r2 : 0.0) / sqrt(x2 > 0.0 ? x2 : 1e-300);
    fits[it - 1] = fit;
    st->iters_done = it;
    const bool last = it >= max_iters;
    const bool conv = fabs(fit - st->prev_fit) < tol;
    st->prev_fit = fit;
    st->skip_update = (it + 1 >= max_iters) ? 1 : 0;
    cudaGraphSetConditional(handle, (last || conv) ? 0u : 1u);
}

__global__ void cpd_state_init_kernel(CpdLoopState *st, const double *x2, int max_iters) {
    st->x2 = *x2;
    st->prev_fit = -1e300;
    st->it = 0;
    st->skip_update = max_iters <= 1 ? 1 : 0;  // the first body run is iteration 1
    st->iters_done = 0;
}

int sm_count() {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms;
}

// partial blocks: >= 256 rows each, at most 2 per SM
int cpd_partial_blocks() { return sm_count() * SYSTEC_CPD_BPS; }

// the ring's dynamic shared-memory opt-in is per device: set before every
// launch (a host-side attribute write), so a plan on any device gets it
template <int RT>
cudaError_t launch_apply_inverse(int PB, size_t rb, cudaStream_t s, const float *M, const float *W, int64_t dim,
                                 int R, float *B, const int *skip, bool ring) {
    // the ring (RT == R) or one synchronously staged tile [kTileRows][RT]
    const size_t smem = ring ? rb : static_cast<size_t>(kTileRows) * RT * 4;
    const cudaError_t attr = cudaFuncSetAttribute(apply_inverse_kernel<RT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                  static_cast<int>(smem));
    if (attr != cudaSuccess) return attr;
    apply_inverse_kernel<RT><<<PB, 256, smem, s>>>(M, W, dim, R, B, skip, ring);
    return cudaSuccess;
}

bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// the tensor-core (3xTF32) forms of the R = 32 dense passes; SYSTEC_CPD_TC=0
// selects the FFMA forms (measurements, A/B)
bool use_tensor_cores() {
    const char *v = std::getenv("SYSTEC_CPD_TC");  // read per call: the tests switch it
    return !(v && v[0] == '0');
}
// the tcgen05 form of the R = 32 pass (cpd_umma.cu) on request
// (SYSTEC_CPD_UMMA=1): correct, but measured slower than the mma.sync form on
// c3 (127 vs 101 us: its 3xTF32 operand copies make it shared-memory bound)
bool use_umma() {
    const char *v = std::getenv("SYSTEC_CPD_UMMA");
    return v && v[0] == '1';
}

// ring form: R % 4 == 0 (contiguous 16-byte rows), R <= 32, 16-byte aligned bases
bool gram_ring(int R, const float *B, const float *M) { return R % 4 == 0 && R <= 32 && aligned16(B) && aligned16(M); }

size_t gram_smem_bytes(int R, bool ring) {
    const size_t tiles = ring ? ring_bytes(2, R) : 2ull * kTileRows * kRp * sizeof(float);
    const size_t redb = (static_cast<size_t>(kRp / 4) * (kRp / 4) * 16 + 256) * sizeof(double);  // row-group sums
    return std::max(tiles, redb);  // ring at R = 32: 96 KB (opt-in dynamic shared-memory limit)
}

// scratch (doubles), in this order:
//   GX[R*R], dots[R]   (contiguous: one reduction) — the pass's G_M and dots
//   GB[R*R]            the Gram of the current (unit-column) iterate, carried
//   H[R*R]             (spare)
//   xhat2[2]           {||Xhat||^2, <X,Xhat>}
//   lam[R], t[R], lt[R], pf[R]  per column: lambda, the stored factor's scale,
//                      W's divisor, the next divisor's correction
//   part[PB][R*R+R]    per-block partials
// floats: W[R*R] (the pass's matrix, F_new = M W)
struct CpdScratch {
    double *GX, *dots, *GB, *H, *xhat2, *part;
    CpdCols cols;
};
CpdScratch layout(double *ds, int R) {
    CpdScratch c;
    c.GX = ds;
    c.dots = c.GX + R * R;
    c.GB = c.dots + R;
    c.H = c.GB + R * R;
    c.xhat2 = c.H + R * R;
    c.cols.lam = c.xhat2 + 2;
    c.cols.t = c.cols.lam + R;
    c.cols.lt = c.cols.t + R;
    c.cols.pf = c.cols.lt + R;
    c.part = c.cols.pf + R;
    return c;
}

int partial_blocks(int64_t dim) {
    return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(cpd_partial_blocks(), (dim + 31) / 32)));
}

// part = per-block {X^T X, column dots X o Y}; then GX, dots = their sums
cudaError_t gram_dots(const float *X, const float *Y, int64_t dim, int R, const CpdScratch &c, cudaStream_t s) {
    const int PB = partial_blocks(dim);
    const int W = R * R + R;
    // R <= 16: warp-shuffle form (c5 14.6 vs 25 us); wider R: the staged
    // register-tile form (R = 32 via shuffles measured 55 vs 27 us: 152
    // registers leave one block per SM)
    if (R <= 8) gram_dots_warp_kernel<8><<<PB, 256, 0, s>>>(X, Y, dim, R, c.part);
    else if (R <= 16) gram_dots_warp_kernel<16><<<PB, 256, 0, s>>>(X, Y, dim, R, c.part);
    else {
        const cudaError_t attr = cudaFuncSetAttribute(  // per device: set at every launch
            gram_dots_partial_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
            static_cast<int>(std::max(gram_smem_bytes(32, true), gram_smem_bytes(kMaxCpR, false))));
        if (attr != cudaSuccess) return attr;
        if (R == 32 && gram_ring(R, X, Y) && use_tensor_cores()) {
            const cudaError_t attr2 = cudaFuncSetAttribute(
                gram_tc32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(gram_smem_bytes(32, true)));
            if (attr2 != cudaSuccess) return attr2;
            gram_tc32_kernel<<<PB, 256, gram_smem_bytes(32, true), s>>>(X, Y, dim, c.part);
        } else if (gram_ring(R, X, Y)) {
            const cudaError_t attr2 = cudaFuncSetAttribute(
                gram_dots_sym_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(gram_smem_bytes(32, true)));
            if (attr2 != cudaSuccess) return attr2;
            gram_dots_sym_kernel<<<PB, 256, gram_smem_bytes(R, true), s>>>(X, Y, dim, R, c.part);
        } else {
            gram_dots_partial_kernel<<<PB, 256, gram_smem_bytes(R, false), s>>>(X, Y, dim, R, c.part);
        }
    }
    reduce_partials_kernel<<<(W + 7) / 8, 256, 0, s>>>(c.part, PB, W, c.GX, nullptr);  // GX and dots (contiguous)
    return cudaGetLastError();
}

// F = M W (skipped when *skip): the FFMA forms
cudaError_t apply_pass(int64_t dim, const float *M, float *F, int R, const float *W, const int *skip, cudaStream_t s) {
    const int PB = partial_blocks(dim);
    // ring form for R in {8, 16, 24, 32} (rows of exactly RT floats), aligned M
    const bool ring = R % 8 == 0 && R <= 32 && aligned16(M);
    const size_t rb = ring ? ring_bytes(1, R) : 0;
    cudaError_t e;
    switch ((R + 7) / 8) {
        case 1: e = launch_apply_inverse<8>(PB, rb, s, M, W, dim, R, F, skip, ring); break;
        case 2: e = launch_apply_inverse<16>(PB, rb, s, M, W, dim, R, F, skip, ring); break;
        case 3: e = launch_apply_inverse<24>(PB, rb, s, M, W, dim, R, F, skip, ring); break;
        case 4: e = launch_apply_inverse<32>(PB, rb, s, M, W, dim, R, F, skip, ring); break;
        case 5: e = launch_apply_inverse<40>(PB, rb, s, M, W, dim, R, F, skip, ring); break;
        default: e = launch_apply_inverse<48>(PB, rb, s, M, W, dim, R, F, skip, ring); break;
    }
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

cudaError_t launch_small(const Plan &p, int R, const CpdScratch &c, float *W, int flags, const int *skip,
                         cudaStream_t s) {
    const size_t smem = small_smem_bytes(R);
    cudaError_t e;
    if (R <= 16) {
        if ((e = cudaFuncSetAttribute(cp_small_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(smem))) != cudaSuccess)
            return e;
        cp_small_kernel<16><<<1, kSmallThreads, smem, s>>>(c.GB, R, p.order, c.cols, c.dots, c.xhat2, c.GX, W, flags, skip);
    } else if (R <= 32) {
        if ((e = cudaFuncSetAttribute(cp_small_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(smem))) != cudaSuccess)
            return e;
        cp_small_kernel<32><<<1, kSmallThreads, smem, s>>>(c.GB, R, p.order, c.cols, c.dots, c.xhat2, c.GX, W, flags, skip);
    } else {
        if ((e = cudaFuncSetAttribute(cp_small_kernel<48>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(smem))) != cudaSuccess)
            return e;
        cp_small_kernel<48><<<1, kSmallThreads, smem, s>>>(c.GB, R, p.order, c.cols, c.dots, c.xhat2, c.GX, W, flags, skip);
    }
    return cudaGetLastError();
}

}  // namespace

int cpd_pass_r32(int form, int64_t dim, const float *M, float *F, const float *W, double *part, int store,
                 const int *skip, cudaStream_t s, cudaError_t *err) {
    *err = cudaSuccess;
    if (form == 1) {
        const cudaError_t e = launch_pass_umma32(M, F, W, dim, part, store, skip, s);
        if (e == cudaSuccess) return cpd_umma_blocks(dim);
        if (e != cudaErrorNotSupported) {
            *err = e;
            return -1;
        }
        cudaGetLastError();  // not available here: the mma.sync form runs
    }
    const int PB = static_cast<int>(
        std::max<int64_t>(1, std::min<int64_t>(static_cast<int64_t>(sm_count()) * kPassBlocksPerSm, (dim + 127) / 128)));
    const size_t smem = ring_bytes<kPassRing>(2, 32);
    cudaError_t e = cudaFuncSetAttribute(pass_tc32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e == cudaSuccess) {
        pass_tc32_kernel<<<PB, kPassThreads, smem, s>>>(M, F, W, dim, part, store, skip);
        e = cudaGetLastError();
    }
    if (e != cudaSuccess) {
        *err = e;
        return -1;
    }
    return PB;
}

int cpd_max_rank() { return kMaxCpR; }

int64_t cpd_scratch_doubles(int R) {
    return 3ll * R * R + 5ll * R + 2 + static_cast<int64_t>(cpd_partial_blocks()) * (R * R + R);
}

int64_t cpd_xhat2_offset(int R) { return 3ll * R * R + R; }

cudaError_t cpd_tensor_norm2(const Plan &p, double *out, cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(out, 0, sizeof(double), s);
    if (e != cudaSuccess || p.nnz == 0) return e;
    const int blocks = sm_count() * 4;
    switch (p.order) {
        case 2: tensor_norm_kernel<2><<<blocks, 256, 0, s>>>(p.coords, p.ld, p.vals, p.nnz, out); break;
        case 3: tensor_norm_kernel<3><<<blocks, 256, 0, s>>>(p.coords, p.ld, p.vals, p.nnz, out); break;
        case 4: tensor_norm_kernel<4><<<blocks, 256, 0, s>>>(p.coords, p.ld, p.vals, p.nnz, out); break;
        case 5: tensor_norm_kernel<5><<<blocks, 256, 0, s>>>(p.coords, p.ld, p.vals, p.nnz, out); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

cudaError_t cpd_init(const Plan &p, const float *B, int R, double *dscratch, float *fscratch, cudaStream_t s) {
    const CpdScratch c = layout(dscratch, R);
    cudaError_t e = gram_dots(B, B, p.dim, R, c, s);  // G_B of the caller's factor (its dots unused)
    if (e != cudaSuccess) return e;
    if ((e = cudaMemcpyAsync(c.GB, c.GX, sizeof(double) * R * R, cudaMemcpyDeviceToDevice, s)) != cudaSuccess) return e;
    cp_cols_init_kernel<<<1, 64, 0, s>>>(c.cols, R);
    return launch_small(p, R, c, fscratch, kSolve, nullptr, s);  // W for iteration 0
}

cudaError_t cpd_step(const Plan &p, const float *M, float *F, int R, double *dscratch, float *fscratch,
                     bool have_lam, bool fit_only, const int *skip, cudaStream_t s) {
    const CpdScratch c = layout(dscratch, R);
    const float *W = fscratch;
    cudaError_t e;
    if (!have_lam) {  // iteration 0: no fit yet
        if (fit_only) return cudaSuccess;
        // two passes: the caller's factor has an arbitrary scale, so lambda_1 is
        // taken from G_M before the apply writes the unit-column B_1
        if ((e = gram_dots(M, F, p.dim, R, c, s)) != cudaSuccess) return e;
        if ((e = launch_small(p, R, c, fscratch, kUpdate | kPrenorm, nullptr, s)) != cudaSuccess) return e;
        if ((e = apply_pass(p.dim, M, F, R, W, nullptr, s)) != cudaSuccess) return e;
        return launch_small(p, R, c, fscratch, kSolve, nullptr, s);
    }
    if ((e = cpd_step_pass(p, M, F, R, dscratch, fscratch, fit_only, skip, s)) != cudaSuccess) return e;
    return cpd_step_algebra(p, R, dscratch, fscratch, fit_only, skip, s);
}

cudaError_t cpd_step_pass(const Plan &p, const float *M, float *F, int R, double *dscratch, const float *fscratch,
                          bool fit_only, const int *skip, cudaStream_t s) {
    const CpdScratch c = layout(dscratch, R);
    const float *W = fscratch;
    cudaError_t e;
    if (R == 32 && gram_ring(R, M, F) && use_tensor_cores()) {
        // the fused pass: G_M, dots M o F and F = M W in one read of M and F
        // (the tcgen05 form when SYSTEC_CPD_UMMA=1 and it can run here)
        const int PB = cpd_pass_r32(use_umma() ? 1 : 0, p.dim, M, F, W, c.part, fit_only ? 0 : 1, skip, s, &e);
        if (PB < 0) return e;
        const int Wd = R * R + R;
        reduce_partials_kernel<<<(Wd + 7) / 8, 256, 0, s>>>(c.part, PB, Wd, c.GX, nullptr);
        return cudaGetLastError();
    }
    if ((e = gram_dots(M, F, p.dim, R, c, s)) != cudaSuccess) return e;  // G_M, dots M o F (the old F)
    if (!fit_only && (e = apply_pass(p.dim, M, F, R, W, skip, s)) != cudaSuccess) return e;
    return cudaSuccess;
}

cudaError_t cpd_step_algebra(const Plan &p, int R, double *dscratch, float *fscratch, bool fit_only, const int *skip,
                             cudaStream_t s) {
    const CpdScratch c = layout(dscratch, R);
    return launch_small(p, R, c, fscratch, kFit | (fit_only ? 0 : kUpdate | kSolve), skip, s);
}

cudaError_t cpd_finish(const Plan &p, float *F, int R, const double *dscratch, float *lam, cudaStream_t s) {
    const CpdScratch c = layout(const_cast<double *>(dscratch), R);
    const int64_t total = p.dim * R;
    const int blocks = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(sm_count() * 8, (total + 255) / 256)));
    cp_finish_kernel<<<blocks, 256, 0, s>>>(F, p.dim, R, c.cols, lam);
    return cudaGetLastError();
}

cudaError_t cpd_state_init(CpdLoopState *st, const double *x2, int max_iters, cudaStream_t s) {
    cpd_state_init_kernel<<<1, 1, 0, s>>>(st, x2, max_iters);
    return cudaGetLastError();
}

cudaError_t cpd_fit_check(const double *dscratch, int R, CpdLoopState *st, double *fits, double tol, int max_iters,
                          cudaGraphConditionalHandle h, cudaStream_t s) {
    const double *xhat2 = dscratch + cpd_xhat2_offset(R);
    cpd_fit_check_kernel<<<1, 1, 0, s>>>(xhat2, st, fits, tol, max_iters, h);
    return cudaGetLastError();
}

}  // namespace systec
