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
// Every step runs in the kernels below (R <= 64; the small R x R algebra in
// one block, in fp64).
#include <algorithm>
#include <cmath>

#include "internal.cuh"

namespace systec {

namespace {

constexpr int kMaxCpR = 48;  // two fp64 R x R tiles + a 256-double scratch in static shared memory

// Two-stage column reductions (no global atomics): each block owns a contiguous
// row range and writes its partial sums; sum_partials_kernel adds the blocks.
//   gram:   part[blk][a*R+b] = sum_{i in blk} B[i][a] B[i][b]       (fp64)
//   coldot: part[blk][r]     = sum_{i in blk} X[i][r] Y[i][r]
__global__ void gram_partial_kernel(const float *__restrict__ B, int64_t dim, int R, double *__restrict__ part) {
    // rows of this block staged in shared memory in tiles, pairs accumulated in fp64
    constexpr int kTileRows = 64;
    __shared__ float tile[kTileRows * kMaxCpR];
    const int64_t rows = (dim + gridDim.x - 1) / gridDim.x;
    const int64_t lo = blockIdx.x * rows, hi = min(dim, lo + rows);
    constexpr int kPairsPerThread = (kMaxCpR * kMaxCpR + 255) / 256;
    double acc[kPairsPerThread];
#pragma unroll
    for (int k = 0; k < kPairsPerThread; ++k) acc[k] = 0.0;
    for (int64_t r0 = lo; r0 < hi; r0 += kTileRows) {
        const int nr = static_cast<int>(min(static_cast<int64_t>(kTileRows), hi - r0));
        __syncthreads();
        for (int q = threadIdx.x; q < nr * R; q += blockDim.x) tile[q] = B[r0 * R + q];
        __syncthreads();
#pragma unroll
        for (int k = 0; k < kPairsPerThread; ++k) {
            const int pidx = threadIdx.x + k * blockDim.x;
            if (pidx < R * R) {
                const int a = pidx / R, b = pidx % R;
                double s0 = 0.0, s1 = 0.0;
                int i = 0;
                for (; i + 1 < nr; i += 2) {
                    s0 += static_cast<double>(tile[i * R + a]) * tile[i * R + b];
                    s1 += static_cast<double>(tile[(i + 1) * R + a]) * tile[(i + 1) * R + b];
                }
                if (i < nr) s0 += static_cast<double>(tile[i * R + a]) * tile[i * R + b];
                acc[k] += s0 + s1;
            }
        }
    }
#pragma unroll
    for (int k = 0; k < kPairsPerThread; ++k) {
        const int pidx = threadIdx.x + k * blockDim.x;
        if (pidx < R * R) part[static_cast<int64_t>(blockIdx.x) * R * R + pidx] = acc[k];
    }
}

__global__ void coldot_partial_kernel(const float *__restrict__ X, const float *__restrict__ Y, int64_t dim, int R,
                                      double *__restrict__ part) {
    const int64_t rows = (dim + gridDim.x - 1) / gridDim.x;
    const int64_t lo = blockIdx.x * rows, hi = min(dim, lo + rows);
    // blockDim = 256: 256/R row lanes x R columns
    const int lanes = blockDim.x / R;
    const int r = threadIdx.x % R, li = threadIdx.x / R;
    __shared__ double red[256];
    double acc = 0.0;
    if (li < lanes)
        for (int64_t i = lo + li; i < hi; i += lanes)
            acc += static_cast<double>(X[i * R + r]) * static_cast<double>(Y[i * R + r]);
    red[threadIdx.x] = (li < lanes) ? acc : 0.0;
    __syncthreads();
    if (threadIdx.x < R) {
        double s = 0.0;
        for (int k = 0; k < lanes; ++k) s += red[k * R + threadIdx.x];
        part[static_cast<int64_t>(blockIdx.x) * R + threadIdx.x] = s;
    }
}

// out[q] = sum_blk part[blk][q], q < width
__global__ void sum_partials_kernel(const double *__restrict__ part, int blocks, int width, double *__restrict__ out) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= width) return;
    double s = 0.0;
    for (int b = 0; b < blocks; ++b) s += part[static_cast<int64_t>(b) * width + q];
    out[q] = s;
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

// One block (blockDim = 256): H = G^{.(n-1)}, Cholesky H = L L^T (tiny relative
// ridge for safety), Hinv = H^{-1}; with lam: ||Xhat||^2 = lam^T G^{.n} lam and
// <X,Xhat> = lam . dots.  Right-looking Cholesky, one column step per barrier.
__global__ void small_solve_kernel(const double *__restrict__ G, int R, int n, float *__restrict__ Hinv,
                                   const float *__restrict__ lam, const double *__restrict__ dots,
                                   double *__restrict__ xhat2) {
    __shared__ double L[kMaxCpR * kMaxCpR];
    __shared__ double Inv[kMaxCpR * kMaxCpR];
    __shared__ double red[256];
    const int tid = threadIdx.x, nt = blockDim.x;
    double fit_part = 0.0;
    for (int p = tid; p < R * R; p += nt) {
        double h = 1.0;
        for (int k = 0; k < n - 1; ++k) h *= G[p];
        L[p] = h;
        if (lam) fit_part += static_cast<double>(lam[p / R]) * lam[p % R] * h * G[p];
    }
    red[tid] = fit_part;
    __syncthreads();
    if (lam && xhat2 && tid == 0) {
        double s = 0.0, ip = 0.0;
        for (int k = 0; k < nt; ++k) s += red[k];
        for (int a = 0; a < R; ++a) ip += static_cast<double>(lam[a]) * dots[a];
        xhat2[0] = s;
        xhat2[1] = ip;
    }
    if (tid == 0) {
        double tr = 0.0;
        for (int a = 0; a < R; ++a) tr += L[a * R + a];
        const double ridge = 1e-12 * (tr / R + 1e-300);
        for (int a = 0; a < R; ++a) L[a * R + a] += ridge;
    }
    __syncthreads();
    for (int j = 0; j < R; ++j) {  // right-looking Cholesky (lower triangle of L)
        if (tid == 0) L[j * R + j] = sqrt(fmax(L[j * R + j], 1e-300));
        __syncthreads();
        const double d = L[j * R + j];
        for (int i = j + 1 + tid; i < R; i += nt) L[i * R + j] /= d;
        __syncthreads();
        for (int p = tid; p < (R - j - 1) * (R - j - 1); p += nt) {
            const int i = j + 1 + p / (R - j - 1), k = j + 1 + p % (R - j - 1);
            if (k <= i) L[i * R + k] -= L[i * R + j] * L[k * R + j];
        }
        __syncthreads();
    }
    // columns of the inverse: solve L L^T x = e_c, one column per thread
    for (int c = tid; c < R; c += nt) {
        double y[kMaxCpR];
        for (int i = 0; i < R; ++i) {
            double sacc = (i == c) ? 1.0 : 0.0;
            for (int k = 0; k < i; ++k) sacc -= L[i * R + k] * y[k];
            y[i] = sacc / L[i * R + i];
        }
        for (int i = R - 1; i >= 0; --i) {
            double sacc = y[i];
            for (int k = i + 1; k < R; ++k) sacc -= L[k * R + i] * Inv[k * R + c];
            Inv[i * R + c] = sacc / L[i * R + i];
        }
    }
    __syncthreads();
    for (int p = tid; p < R * R; p += nt) Hinv[p] = static_cast<float>(Inv[p]);
}

// Bout[i][b] = sum_a M[i][a] Hinv[a][b]
__global__ void apply_inverse_kernel(const float *__restrict__ M, const float *__restrict__ Hinv, int64_t dim, int R,
                                     float *__restrict__ Bout) {
    __shared__ float Hs[kMaxCpR * kMaxCpR];
    for (int p = threadIdx.x; p < R * R; p += blockDim.x) Hs[p] = Hinv[p];
    __syncthreads();
    const int64_t total = dim * R;
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = q / R;
        const int b = static_cast<int>(q % R);
        float s = 0.f;
        for (int a = 0; a < R; ++a) s += M[i * R + a] * Hs[a * R + b];
        Bout[q] = s;
    }
}

// lam[b] = sqrt(norms[b]); B[i][b] /= lam[b]
__global__ void normalize_kernel(float *__restrict__ B, int64_t dim, int R, const double *__restrict__ norms,
                                 float *__restrict__ lam) {
    const int64_t total = dim * R;
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
        const int b = static_cast<int>(q % R);
        const double nb = sqrt(norms[b]);
        B[q] = nb > 0 ? static_cast<float>(B[q] / nb) : B[q];
    }
    if (blockIdx.x == 0)
        for (int b = threadIdx.x; b < R; b += blockDim.x) lam[b] = static_cast<float>(sqrt(norms[b]));
}

int sm_count() {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms;
}

}  // namespace

int cpd_max_rank() { return kMaxCpR; }

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

int cpd_partial_blocks() { return sm_count() * 4; }

// scratch (doubles): G[R*R], dots[R], norms[R], scalars[2] = {||Xhat||^2, <X,Xhat>},
// then partials[PB][R*R] | floats: Hinv[R*R]
int64_t cpd_scratch_doubles(int R) { return static_cast<int64_t>(R) * R + 2 * R + 2 + static_cast<int64_t>(cpd_partial_blocks()) * R * R; }

cudaError_t cpd_step(const Plan &p, const float *M, float *B, float *lam, int R, double *dscratch,
                     float *fscratch, bool have_lam, bool fit_only, cudaStream_t s) {
    double *G = dscratch, *dots = G + R * R, *norms = dots + R, *xhat2 = norms + R, *part = xhat2 + 2;
    float *Hinv = fscratch;
    // partial blocks: ~128 rows each, at most 4 per SM
    const int PB = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(cpd_partial_blocks(), (p.dim + 127) / 128)));
    const int rr = R * R;
    gram_partial_kernel<<<PB, 256, 0, s>>>(B, p.dim, R, part);
    sum_partials_kernel<<<(rr + 255) / 256, 256, 0, s>>>(part, PB, rr, G);
    coldot_partial_kernel<<<PB, 256, 0, s>>>(M, B, p.dim, R, part);   // <X,Xhat> pieces of the current iterate
    sum_partials_kernel<<<1, 64, 0, s>>>(part, PB, R, dots);
    small_solve_kernel<<<1, 256, 0, s>>>(G, R, p.order, Hinv, have_lam ? lam : nullptr, dots, xhat2);
    if (fit_only) return cudaGetLastError();
    const int64_t total = p.dim * R;
    const int ab = static_cast<int>(std::min<int64_t>((total + 255) / 256, static_cast<int64_t>(sm_count()) * 8));
    apply_inverse_kernel<<<ab, 256, 0, s>>>(M, Hinv, p.dim, R, B);
    coldot_partial_kernel<<<PB, 256, 0, s>>>(B, B, p.dim, R, part);   // squared column norms of B_new
    sum_partials_kernel<<<1, 64, 0, s>>>(part, PB, R, norms);
    normalize_kernel<<<ab, 256, 0, s>>>(B, p.dim, R, norms, lam);
    return cudaGetLastError();
}

}  // namespace systec
