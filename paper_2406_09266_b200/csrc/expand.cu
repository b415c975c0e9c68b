// expand.cu — materialise the non-symmetric tensor a symmetric one stands for:
// every stored entry becomes all DISTINCT permutations of its indices (the
// orbit of Def. Symmetry; n!/prod m! members,
// PAPER.md:289-291).  This is the input of the non-symmetric baseline kernel
// (the paper's "naive" comparison).
#include <cub/device/device_scan.cuh>

#include "internal.cuh"

namespace systec {

namespace {

template <int N>
__device__ __forceinline__ void sort_small(int32_t (&c)[N]) {
#pragma unroll
    for (int r = 0; r < N; ++r) {
#pragma unroll
        for (int t = r & 1; t + 1 < N; t += 2) {
            const int32_t a = c[t], b = c[t + 1];
            c[t] = min(a, b);
            c[t + 1] = max(a, b);
        }
    }
}

// lexicographic successor of a multiset permutation; false after the last one
template <int N>
__device__ __forceinline__ bool next_perm(int32_t (&p)[N]) {
    int i = N - 2;
    while (i >= 0 && p[i] >= p[i + 1]) --i;
    if (i < 0) return false;
    int j = N - 1;
    while (p[j] <= p[i]) --j;
    int32_t t = p[i];
    p[i] = p[j];
    p[j] = t;
    for (int a = i + 1, b = N - 1; a < b; ++a, --b) {
        t = p[a];
        p[a] = p[b];
        p[b] = t;
    }
    return true;
}

template <int N>
__global__ void orbit_size_kernel(const int32_t *__restrict__ idx, int64_t nnz, int64_t dim,
                                  unsigned long long *__restrict__ sizes, DevStats *st) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x) {
        int32_t c[N];
        bool ok = true;
#pragma unroll
        for (int t = 0; t < N; ++t) {
            c[t] = idx[e * N + t];
            ok &= (c[t] >= 0) & (static_cast<int64_t>(c[t]) < dim);
        }
        if (!ok) {
            atomicOr(&st->err, 1ull);
            atomicMin(&st->bad_entry, static_cast<unsigned long long>(e));
            sizes[e] = 0;
            continue;
        }
        sort_small<N>(c);
        unsigned long long n = 0;
        do { ++n; } while (next_perm<N>(c));
        sizes[e] = n;
    }
}

template <int N>
__global__ void expand_kernel(const int32_t *__restrict__ idx, const float *__restrict__ vals, int64_t nnz,
                              const unsigned long long *__restrict__ offsets, int32_t *__restrict__ out_idx,
                              float *__restrict__ out_vals) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x) {
        int32_t c[N];
#pragma unroll
        for (int t = 0; t < N; ++t) c[t] = idx[e * N + t];
        sort_small<N>(c);
        const float v = vals[e];
        unsigned long long o = offsets[e];
        do {
#pragma unroll
            for (int t = 0; t < N; ++t) out_idx[o * N + t] = c[t];
            out_vals[o] = v;
            ++o;
        } while (next_perm<N>(c));
    }
}

int grid_of(int64_t n) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t want = (n + 255) / 256;
    return static_cast<int>(want < 1 ? 1 : (want > sms * 16ll ? sms * 16ll : want));
}

}  // namespace

#define SYSTEC_ORDER_SWITCH2(order, ...)                     \
    switch (order) {                                          \
        case 2: { constexpr int N = 2; __VA_ARGS__; } break; \
        case 3: { constexpr int N = 3; __VA_ARGS__; } break; \
        case 4: { constexpr int N = 4; __VA_ARGS__; } break; \
        case 5: { constexpr int N = 5; __VA_ARGS__; } break; \
        default: return cudaErrorInvalidValue;                \
    }

cudaError_t expand_count(int order, int64_t dim, int64_t nnz, const int32_t *idx, unsigned long long *sizes,
                         unsigned long long *offsets, DevStats *st, cudaStream_t s) {
    if (nnz == 0) return cudaSuccess;
    SYSTEC_ORDER_SWITCH2(order, orbit_size_kernel<N><<<grid_of(nnz), 256, 0, s>>>(idx, nnz, dim, sizes, st));
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    size_t temp = 0;
    e = cub::DeviceScan::ExclusiveSum(nullptr, temp, sizes, offsets, static_cast<int>(nnz), s);
    if (e != cudaSuccess) return e;
    void *tmp = nullptr;
    if ((e = cudaMallocAsync(&tmp, temp ? temp : 16, s)) != cudaSuccess) return e;
    e = cub::DeviceScan::ExclusiveSum(tmp, temp, sizes, offsets, static_cast<int>(nnz), s);
    cudaError_t f = cudaFreeAsync(tmp, s);
    return e != cudaSuccess ? e : f;
}

cudaError_t expand_write(int order, int64_t nnz, const int32_t *idx, const float *vals,
                         const unsigned long long *offsets, int32_t *out_idx, float *out_vals, cudaStream_t s) {
    if (nnz == 0) return cudaSuccess;
    SYSTEC_ORDER_SWITCH2(order, expand_kernel<N><<<grid_of(nnz), 256, 0, s>>>(idx, vals, nnz, offsets, out_idx, out_vals));
    return cudaGetLastError();
}

}  // namespace systec
