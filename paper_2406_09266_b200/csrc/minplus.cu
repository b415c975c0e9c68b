// minplus.cu — one Bellman-Ford relaxation over a symmetric sparse matrix in
// the (min, +) semiring (the paper's Bellman-Ford
// kernel `y[i] min= A[i,j] + d[j]`, "identical to SSYMV").
//
// A stored canonical entry (i <= j; v) stands for A[i,j] = A[j,i] = v
// (Def. Symmetry).  Min is idempotent, so the distributive
// grouping of PAPER.md:577-591 collapses repeated updates to ONE (no
// multiplicity factor): the entry updates
//     y[i] = min(y[i], v + d[j])   and, if i != j,   y[j] = min(y[j], v + d[i]).
// The output starts at y = d (one relaxation step).  Arithmetic is fp32: each
// candidate v + d is one rounded add, the min is exact — so the result is
// independent of the order of the atomic updates (bit-exact).
//
// Mapping: each warp takes a contiguous range of the sorted stream; lane = one
// entry; equal leading indices are contiguous, so a segmented warp min-scan
// gives one atomic per run of i per 32 entries; the j updates go straight to an
// order-preserving integer atomicMin.
#include <algorithm>
#include <cfloat>
#include <climits>

#include "internal.cuh"

namespace systec {

namespace {

// float -> int order-preserving key (monotone for all non-NaN floats)
__device__ __forceinline__ int fkey(float f) {
    const int b = __float_as_int(f);
    return b >= 0 ? b : b ^ 0x7fffffff;
}
__device__ __forceinline__ float unkey(int k) { return __int_as_float(k >= 0 ? k : k ^ 0x7fffffff); }

__global__ void minplus_init_kernel(const float *__restrict__ d, int *__restrict__ ykey, int64_t dim) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < dim; i += (int64_t)gridDim.x * blockDim.x)
        ykey[i] = fkey(d[i]);
}

__global__ void minplus_finish_kernel(const int *__restrict__ ykey, float *__restrict__ y, int64_t dim) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < dim; i += (int64_t)gridDim.x * blockDim.x)
        y[i] = unkey(ykey[i]);
}

__global__ void __launch_bounds__(256) minplus_sym2_kernel(const int32_t *__restrict__ c0, const int32_t *__restrict__ c1,
                                                           const float *__restrict__ vals, int64_t nnz, int64_t span,
                                                           const float *__restrict__ d, int *__restrict__ ykey) {
    const int lane = threadIdx.x & 31;
    const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t begin = gw * span;
    const int64_t end = min(begin + span, nnz);
    for (int64_t base = begin; base < end; base += 32) {
        const int64_t e = base + lane;
        const bool ok = e < end;
        int i = -1, j = -1;
        float v = 0.f;
        if (ok) {
            i = __ldg(c0 + e);
            j = __ldg(c1 + e);
            v = __ldg(vals + e);
        }
        int ki = ok ? fkey(v + __ldg(d + j)) : INT_MAX;  // candidate for y[i]
        if (ok && i != j) atomicMin(ykey + j, fkey(v + __ldg(d + i)));
        // segmented min over lanes with equal i (contiguous: the stream is sorted)
#pragma unroll
        for (int s = 1; s < 32; s <<= 1) {
            const int oi = __shfl_down_sync(0xffffffffu, i, s);
            const int ok2 = __shfl_down_sync(0xffffffffu, ki, s);
            if (lane + s < 32 && oi == i) ki = min(ki, ok2);
        }
        const int pi = __shfl_up_sync(0xffffffffu, i, 1);
        if (ok && (lane == 0 || pi != i)) atomicMin(ykey + i, ki);
    }
}

__global__ void sssp_init_kernel(float *__restrict__ d, int64_t dim, int64_t source) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < dim; i += (int64_t)gridDim.x * blockDim.x)
        d[i] = (i == source) ? 0.f : __int_as_float(0x7f800000);  // +inf
}

// d = y where they differ, *changed |= any difference (one pass: the
// relaxation's convergence test and the copy back together)
__global__ void sssp_update_kernel(const float *__restrict__ y, float *__restrict__ d, int64_t dim, int *changed) {
    bool any = false;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < dim; i += (int64_t)gridDim.x * blockDim.x) {
        const float v = y[i];
        if (v != d[i]) {
            d[i] = v;
            any = true;
        }
    }
    if (__any_sync(0xffffffffu, any) && (threadIdx.x & 31) == 0) atomicOr(changed, 1);
}

// device-side loop control of the SSSP graph: one more relaxation while
// something changed and the iteration budget lasts
__global__ void sssp_step_kernel(const int *changed, int *iters, int max_iters, cudaGraphConditionalHandle h) {
    const int it = ++(*iters);
    cudaGraphSetConditional(h, (*changed != 0 && it < max_iters) ? 1u : 0u);
}

}  // namespace

cudaError_t launch_sssp_update(const float *y, float *d, int64_t dim, int *changed, cudaStream_t s) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int gb = static_cast<int>(std::min<int64_t>((dim + 255) / 256, static_cast<int64_t>(sms) * 8));
    cudaError_t e = cudaMemsetAsync(changed, 0, sizeof(int), s);
    if (e != cudaSuccess) return e;
    sssp_update_kernel<<<gb, 256, 0, s>>>(y, d, dim, changed);
    return cudaGetLastError();
}

cudaError_t launch_sssp_step(const int *changed, int *iters, int max_iters, cudaGraphConditionalHandle h,
                             cudaStream_t s) {
    sssp_step_kernel<<<1, 1, 0, s>>>(changed, iters, max_iters, h);
    return cudaGetLastError();
}

cudaError_t launch_sssp_init(float *d, int64_t dim, int64_t source, cudaStream_t s) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int gb = static_cast<int>(std::min<int64_t>((dim + 255) / 256, static_cast<int64_t>(sms) * 8));
    sssp_init_kernel<<<gb, 256, 0, s>>>(d, dim, source);
    return cudaGetLastError();
}

cudaError_t launch_minplus(const Plan &p, const float *d, float *y, int *scratch_keys, cudaStream_t s) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int th = 256;
    const int gb = static_cast<int>(std::min<int64_t>((p.dim + th - 1) / th, static_cast<int64_t>(sms) * 8));
    minplus_init_kernel<<<gb, th, 0, s>>>(d, scratch_keys, p.dim);
    if (p.nnz > 0) {
        const int64_t warps = static_cast<int64_t>(sms) * 64;
        int64_t span = (p.nnz + warps - 1) / warps;
        span = ((span + 31) / 32) * 32;
        const int64_t blocks = ((p.nnz + span - 1) / span + 7) / 8;
        minplus_sym2_kernel<<<static_cast<unsigned>(blocks), th, 0, s>>>(p.coords, p.coords + p.ld, p.vals, p.nnz,
                                                                         span, d, scratch_keys);
    }
    minplus_finish_kernel<<<gb, th, 0, s>>>(scratch_keys, y, p.dim);
    return cudaGetLastError();
}

}  // namespace systec
