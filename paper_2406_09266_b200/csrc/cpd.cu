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

constexpr int kMaxCpR = 48;  // two fp64 R x R tiles in static shared memory

// G[a][b] += sum over this block's rows of B[i][a] * B[i][b]   (fp64 accumulation)
__global__ void gram_kernel(const float *__restrict__ B, int64_t dim, int R, double *__restrict__ G) {
    const int pairs = R * R;
    for (int pidx = threadIdx.x; pidx < pairs; pidx += blockDim.x) {
        const int a = pidx / R, b = pidx % R;
        double acc = 0.0;
        for (int64_t i = blockIdx.x; i < dim; i += gridDim.x)
            acc += static_cast<double>(B[i * R + a]) * static_cast<double>(B[i * R + b]);
        atomicAdd(&G[pidx], acc);
    }
}

// w[r] += sum_i X[i][r] * Y[i][r]
__global__ void coldot_kernel(const float *__restrict__ X, const float *__restrict__ Y, int64_t dim, int R,
                              double *__restrict__ w) {
    for (int r = threadIdx.x; r < R; r += blockDim.x) {
        double acc = 0.0;
        for (int64_t i = blockIdx.x; i < dim; i += gridDim.x)
            acc += static_cast<double>(X[i * R + r]) * static_cast<double>(Y[i * R + r]);
        atomicAdd(&w[r], acc);
    }
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

// One block: H = G^{.(n-1)}, Cholesky H = L L^T (with a tiny relative ridge
// for safety), Hinv = H^{-1}; also ||Xhat||^2 = lam^T G^{.n} lam when lam given.
__global__ void small_solve_kernel(const double *__restrict__ G, int R, int n, float *__restrict__ Hinv,
                                   const float *__restrict__ lam, const double *__restrict__ dots,
                                   double *__restrict__ xhat2) {
    __shared__ double L[kMaxCpR * kMaxCpR];
    __shared__ double Inv[kMaxCpR * kMaxCpR];
    const int tid = threadIdx.x;
    for (int p = tid; p < R * R; p += blockDim.x) {
        double h = 1.0;
        for (int k = 0; k < n - 1; ++k) h *= G[p];
        L[p] = h;
    }
    __syncthreads();
    if (tid == 0) {
        if (lam && xhat2) {  // fit pieces of the current iterate: ||Xhat||^2 and <X, Xhat>
            double s = 0.0;
            for (int a = 0; a < R; ++a)
                for (int b = 0; b < R; ++b) {
                    double g = 1.0;
                    for (int k = 0; k < n; ++k) g *= G[a * R + b];
                    s += static_cast<double>(lam[a]) * lam[b] * g;
                }
            xhat2[0] = s;
            double ip = 0.0;
            for (int a = 0; a < R; ++a) ip += static_cast<double>(lam[a]) * dots[a];
            xhat2[1] = ip;
        }
        double tr = 0.0;
        for (int a = 0; a < R; ++a) tr += L[a * R + a];
        const double ridge = 1e-12 * (tr / R + 1e-300);
        for (int a = 0; a < R; ++a) L[a * R + a] += ridge;
        // in-place Cholesky (lower)
        for (int j = 0; j < R; ++j) {
            double d = L[j * R + j];
            for (int k = 0; k < j; ++k) d -= L[j * R + k] * L[j * R + k];
            d = sqrt(fmax(d, 1e-300));
            L[j * R + j] = d;
            for (int i = j + 1; i < R; ++i) {
                double s = L[i * R + j];
                for (int k = 0; k < j; ++k) s -= L[i * R + k] * L[j * R + k];
                L[i * R + j] = s / d;
            }
        }
    }
    __syncthreads();
    // columns of the inverse: solve L L^T x = e_c, one column per thread
    for (int c = tid; c < R; c += blockDim.x) {
        double y[kMaxCpR];
        for (int i = 0; i < R; ++i) {
            double s = (i == c) ? 1.0 : 0.0;
            for (int k = 0; k < i; ++k) s -= L[i * R + k] * y[k];
            y[i] = s / L[i * R + i];
        }
        for (int i = R - 1; i >= 0; --i) {
            double s = y[i];
            for (int k = i + 1; k < R; ++k) s -= L[k * R + i] * Inv[k * R + c];
            Inv[i * R + c] = s / L[i * R + i];
        }
    }
    __syncthreads();
    for (int p = tid; p < R * R; p += blockDim.x) Hinv[p] = static_cast<float>(Inv[p]);
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

// scratch layout (doubles): G[R*R], dots[R], norms[R], scalars[2] = {||Xhat||^2, <X,Xhat>} | floats: Hinv[R*R]
cudaError_t cpd_step(const Plan &p, const float *M, float *B, float *lam, int R, double *dscratch,
                     float *fscratch, bool have_lam, bool fit_only, cudaStream_t s) {
    double *G = dscratch, *dots = G + R * R, *norms = dots + R, *xhat2 = norms + R;
    float *Hinv = fscratch;
    cudaError_t e = cudaMemsetAsync(dscratch, 0, sizeof(double) * (R * R + 2 * R + 2), s);
    if (e != cudaSuccess) return e;
    const int blocks = std::max(1, std::min(sm_count() * 4, static_cast<int>((p.dim + 63) / 64)));
    gram_kernel<<<blocks, 256, 0, s>>>(B, p.dim, R, G);
    coldot_kernel<<<blocks, 64, 0, s>>>(M, B, p.dim, R, dots);     // <X,Xhat> pieces for the current iterate
    small_solve_kernel<<<1, 64, 0, s>>>(G, R, p.order, Hinv, have_lam ? lam : nullptr, dots, xhat2);
    if (fit_only) return cudaGetLastError();
    const int64_t total = p.dim * R;
    const int ab = static_cast<int>(std::min<int64_t>((total + 255) / 256, static_cast<int64_t>(sm_count()) * 8));
    apply_inverse_kernel<<<ab, 256, 0, s>>>(M, Hinv, p.dim, R, B);
    coldot_kernel<<<blocks, 64, 0, s>>>(B, B, p.dim, R, norms);     // squared column norms of B_new
    normalize_kernel<<<ab, 256, 0, s>>>(B, p.dim, R, norms, lam);
    return cudaGetLastError();
}

}  // namespace systec
