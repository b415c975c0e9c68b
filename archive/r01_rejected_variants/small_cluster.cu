// small.cu — one-launch path for small problems (latency-bound sizes such as
// c1: 2,000 entries, a 2 KB output).  At these sizes the main path's fixed
// costs dominate: a C memset launch, the per-warp mbarrier/TMA set-up, and a
// chain of dependent HBM round trips.  This path is ONE launch of ONE thread-
// block cluster (8 CTAs x 1024 threads): every CTA accumulates its share of
// the entries into a private copy of C in shared memory, the cluster syncs,
// and each CTA sums one slice of C across the 8 copies through distributed
// shared memory (DSMEM) and writes it to C.  No memset, no global atomics, no
// scratch.  Arithmetic is the main kernel's (paper Listing 6 / Sec. 4.3): per
// stored entry and run-first position t,
//   C[c_t, r] += coef_t(pattern) * v * prod_{s != t} B[c_s, r].
#include <algorithm>
#include <cooperative_groups.h>

#include "coef_table.cuh"
#include "internal.cuh"

namespace cg = cooperative_groups;

namespace systec {

namespace {

constexpr int kSmallCtas = 8;       // one portable cluster
constexpr int kSmallThreads = 1024;

static __constant__ CoefTable kCoefSmall = make_coef_table();

__device__ __forceinline__ float4 mul4(float4 a, float4 b) {
    return make_float4(a.x * b.x, a.y * b.y, a.z * b.z, a.w * b.w);
}

// VW = 4: one thread per (entry, float4 column group); VW = 1: per (entry, column).
template <int N, int VW>
__global__ void __cluster_dims__(kSmallCtas, 1, 1) __launch_bounds__(kSmallThreads)
    mttkrp_small_kernel(const int32_t *__restrict__ coords, int64_t ld, const float *__restrict__ vals, int64_t nnz,
                        const float *__restrict__ B, int R, int plane, float *__restrict__ C, int accumulate) {
    extern __shared__ float4 smem4[];
    float *Cs = reinterpret_cast<float *>(smem4);
    cg::cluster_group cluster = cg::this_cluster();
    const int rank = static_cast<int>(cluster.block_rank());
    for (int q = threadIdx.x; q < plane; q += blockDim.x) Cs[q] = 0.f;
    __syncthreads();

    const int vecs = R / VW;
    const int64_t items = nnz * vecs;
    for (int64_t w = static_cast<int64_t>(rank) * blockDim.x + threadIdx.x; w < items;
         w += static_cast<int64_t>(kSmallCtas) * blockDim.x) {
        const int64_t e = w / vecs;
        const int col = static_cast<int>(w - e * vecs) * VW;
        int32_t c[N];
#pragma unroll
        for (int t = 0; t < N; ++t) c[t] = __ldg(coords + t * ld + e);
        const float v = __ldg(vals + e);
        int code = 0;
#pragma unroll
        for (int t = 0; t + 1 < N; ++t) code |= (c[t] == c[t + 1]) << t;
        const float *cf = kCoefSmall.v[N - 2][code];
        if constexpr (VW == 4) {
            float4 b[N];
#pragma unroll
            for (int t = 0; t < N; ++t) b[t] = __ldg(reinterpret_cast<const float4 *>(B + static_cast<int64_t>(c[t]) * R + col));
#pragma unroll
            for (int t = 0; t < N; ++t) {
                const float k = cf[t] * v;
                if (k == 0.f) continue;
                float4 prod = make_float4(k, k, k, k);
#pragma unroll
                for (int s2 = 0; s2 < N; ++s2)
                    if (s2 != t) prod = mul4(prod, b[s2]);
                float *dst = Cs + c[t] * R + col;
                atomicAdd(dst + 0, prod.x);
                atomicAdd(dst + 1, prod.y);
                atomicAdd(dst + 2, prod.z);
                atomicAdd(dst + 3, prod.w);
            }
        } else {
            float b[N];
#pragma unroll
            for (int t = 0; t < N; ++t) b[t] = __ldg(B + static_cast<int64_t>(c[t]) * R + col);
#pragma unroll
            for (int t = 0; t < N; ++t) {
                float prod = cf[t] * v;
                if (prod == 0.f) continue;
#pragma unroll
                for (int s2 = 0; s2 < N; ++s2)
                    if (s2 != t) prod *= b[s2];
                atomicAdd(Cs + c[t] * R + col, prod);
            }
        }
    }
    cluster.sync();  // every CTA's private C complete and visible cluster-wide

    // CTA `rank` owns a contiguous slice of C; sum it over the 8 copies (DSMEM)
    const float *peer[kSmallCtas];
#pragma unroll
    for (int r2 = 0; r2 < kSmallCtas; ++r2) peer[r2] = cluster.map_shared_rank(Cs, r2);
    if constexpr (VW == 4) {
        const int nv = plane / 4;
        const int per = (nv + kSmallCtas - 1) / kSmallCtas;
        const int lo = rank * per, hi = min(nv, lo + per);
        for (int q = lo + threadIdx.x; q < hi; q += blockDim.x) {
            float4 acc = accumulate ? reinterpret_cast<const float4 *>(C)[q] : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int r2 = 0; r2 < kSmallCtas; ++r2) {
                const float4 x = reinterpret_cast<const float4 *>(peer[r2])[q];
                acc.x += x.x; acc.y += x.y; acc.z += x.z; acc.w += x.w;
            }
            reinterpret_cast<float4 *>(C)[q] = acc;
        }
    } else {
        const int per = (plane + kSmallCtas - 1) / kSmallCtas;
        const int lo = rank * per, hi = min(plane, lo + per);
        for (int q = lo + threadIdx.x; q < hi; q += blockDim.x) {
            float acc = accumulate ? C[q] : 0.f;
#pragma unroll
            for (int r2 = 0; r2 < kSmallCtas; ++r2) acc += peer[r2][q];
            C[q] = acc;
        }
    }
    cluster.sync();  // keep every CTA's shared memory alive until the peers have read it
}

template <int N, int VW>
cudaError_t launch_small_t(const Plan &p, const float *B, int R, float *C, int plane, bool acc, cudaStream_t s) {
    const size_t smem = static_cast<size_t>(plane) * 4;
    auto fn = mttkrp_small_kernel<N, VW>;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        if (e != cudaSuccess) return e;
    }
    fn<<<kSmallCtas, kSmallThreads, smem, s>>>(p.coords, p.ld, p.vals, p.nnz, B, R, plane, C, acc ? 1 : 0);
    return cudaGetLastError();
}

}  // namespace

int64_t small_path_max_items() { return 32768; }
int64_t small_path_max_plane() { return 24 * 1024; }  // floats of C (96 KB of shared memory per CTA)

// One-cluster path.  Returns cudaErrorNotSupported when the problem is outside
// its range (the caller then takes the main path).
cudaError_t launch_mttkrp_small(Plan &p, const float *B, int R, float *C, bool accumulate, cudaStream_t s) {
    const int64_t plane = p.dim * static_cast<int64_t>(R);
    if (p.general || p.nnz == 0 || p.order < 2 || p.order > 5 || plane > small_path_max_plane())
        return cudaErrorNotSupported;
    const bool aligned = (reinterpret_cast<uintptr_t>(B) % 16 == 0) && (reinterpret_cast<uintptr_t>(C) % 16 == 0);
    const int vw = (R % 4 == 0 && aligned) ? 4 : 1;
    if (p.nnz * (R / vw) > small_path_max_items()) return cudaErrorNotSupported;
    const int ip = static_cast<int>(plane);
    cudaError_t e;
    switch (p.order * 10 + vw) {
        case 24: e = launch_small_t<2, 4>(p, B, R, C, ip, accumulate, s); break;
        case 21: e = launch_small_t<2, 1>(p, B, R, C, ip, accumulate, s); break;
        case 34: e = launch_small_t<3, 4>(p, B, R, C, ip, accumulate, s); break;
        case 31: e = launch_small_t<3, 1>(p, B, R, C, ip, accumulate, s); break;
        case 44: e = launch_small_t<4, 4>(p, B, R, C, ip, accumulate, s); break;
        case 41: e = launch_small_t<4, 1>(p, B, R, C, ip, accumulate, s); break;
        case 54: e = launch_small_t<5, 4>(p, B, R, C, ip, accumulate, s); break;
        default: e = launch_small_t<5, 1>(p, B, R, C, ip, accumulate, s); break;
    }
    p.last_grid_x = kSmallCtas;
    p.last_grid_y = 1;
    p.last_block = kSmallThreads;
    p.last_smem = ip * 4;
    p.last_kernel = 2000000000 + p.order * 100000 + vw * 10000;  // small path: 2 | order | vw
    return e;
}

}  // namespace systec
