// sym2_window.cu — order-2 symmetric SpMM / SpMV without atomics (SURVEY.md
// §8(f) NEXT-3: SSYMV / SSYMM).
//
// A symmetric matrix is stored once, as its canonical upper triangle
// (i <= j), sorted by row.  Each stored entry stands for two updates
// (PAPER.md Listing for SSYMV: y[i] += A[i,j] x[j]; y[j] += A[i,j] x[i]).  The
// general kernel (mttkrp_kernel.cuh) accumulates the first along the row and
// issues a red.global for the second — one L2 atomic per stored entry, which
// on the B200 costs ~2.5x a row gather (6 vs 15 TB/s of 128-B rows), so at
// R = 32 it loses to the naive kernel over both triangles.
//
// This kernel takes the transposed updates off the atomics.  The rows are
// cut into blocks of <= 768 rows whose column lists fit in shared memory;
// one CTA per block:
//   1. reads the stream segment of its rows AND the `bw` rows above them
//      (bw = max(j - i), the matrix bandwidth: every entry (i, j) with j in
//      the block has i >= r0 - bw), and scatters each entry with j in the
//      block into a shared-memory column list of row j (item = (i, v));
//      positions come from the plan's column pointer (the upper triangle's
//      CSC counts, built at plan creation) plus a shared-memory cursor;
//   2. computes every row q of the block completely in registers —
//      C[q] = sum_{(q,j) stored} v B[j] + sum_{(i,q) stored, i<q} v B[i] — and
//      writes it with ONE plain store (no atomics, no zeroing pass).
// Each stored entry is read once from HBM (plus the bw-row halo, re-read by
// the next block) and yields both of its updates: the paper's "one read,
// several updates" moved into on-chip memory.  Used for
// low-bandwidth matrices (bw <= the mean block height), the structure of
// the FEM / structural matrices of the paper's SSYMV suite; other order-2
// plans keep the general kernel.
#include <cub/cub.cuh>

#include "internal.cuh"
#include "ptx.cuh"

namespace systec {

namespace {

constexpr int kWinCap = 4608;                   // column-list items per block (8 B each: 36 KB)
constexpr int kWinRowW = 6;                     // row weight in the partition
constexpr int kWinMaxRows = kWinCap / kWinRowW;  // <= 768 rows per block

// rowptr[q] = first stored entry with c0 >= q, q in [0, dim]
__global__ void win_rowptr_kernel(const int32_t *__restrict__ c0, int64_t nnz, int64_t dim, int32_t *__restrict__ rowptr) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e <= nnz; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t lo = e == 0 ? -1 : c0[e - 1];
        const int64_t hi = e == nnz ? dim : c0[e];
        for (int64_t q = lo + 1; q <= hi; ++q) rowptr[q] = static_cast<int32_t>(e);
    }
}

// colcnt[j] += 1 per off-diagonal stored entry (i, j); bw = max(j - i)
__global__ void win_colcount_kernel(const int32_t *__restrict__ c0, const int32_t *__restrict__ c1, int64_t nnz,
                                    int32_t *__restrict__ colcnt, unsigned long long *__restrict__ bw) {
    unsigned long long m = 0;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x) {
        const int32_t i = c0[e], j = c1[e];
        if (i != j) atomicAdd(&colcnt[j], 1);
        m = max(m, static_cast<unsigned long long>(j - i));
    }
#pragma unroll
    for (int d = 16; d; d >>= 1) m = max(m, __shfl_down_sync(0xffffffffu, m, d));
    if ((threadIdx.x & 31) == 0 && m) atomicMax(bw, m);
}

__global__ void win_maxcol_kernel(const int32_t *__restrict__ colcnt, int64_t dim, unsigned long long *__restrict__ mx) {
    unsigned long long m = 0;
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < dim; q += (int64_t)gridDim.x * blockDim.x)
        m = max(m, static_cast<unsigned long long>(colcnt[q]));
#pragma unroll
    for (int d = 16; d; d >>= 1) m = max(m, __shfl_down_sync(0xffffffffu, m, d));
    if ((threadIdx.x & 31) == 0 && m) atomicMax(mx, m);
}

struct WinParams {
    const int32_t *c0, *c1;
    const float *vals;
    const int32_t *rowptr, *colptr;  // [dim + 1] each
    const float *B;
    float *C;
    int64_t dim;
    int bw;
    int capp;   // partition step: kWinCap - (max column count + kWinRowW)
    int nblk;
    int R;
};

// first q in [0, dim] with colptr[q] + kWinRowW * q >= x
__device__ int win_lower(const WinParams &p, int64_t x) {
    int64_t lo = 0, hi = p.dim;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (static_cast<int64_t>(p.colptr[mid]) + kWinRowW * mid >= x) hi = mid;
        else lo = mid + 1;
    }
    return static_cast<int>(lo);
}

template <int VW> struct WinVec;
template <> struct WinVec<4> {
    using T = float4;
    static __device__ __forceinline__ T zero() { return make_float4(0.f, 0.f, 0.f, 0.f); }
    static __device__ __forceinline__ T load(const float *p) { return __ldg(reinterpret_cast<const float4 *>(p)); }
    static __device__ __forceinline__ T fma(float v, T b, T a) {
        return make_float4(fmaf(v, b.x, a.x), fmaf(v, b.y, a.y), fmaf(v, b.z, a.z), fmaf(v, b.w, a.w));
    }
    static __device__ __forceinline__ T add(T a, T b) { return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w); }
    static __device__ __forceinline__ void store(float *p, T v) { *reinterpret_cast<float4 *>(p) = v; }
};
template <> struct WinVec<1> {
    using T = float;
    static __device__ __forceinline__ T zero() { return 0.f; }
    static __device__ __forceinline__ T load(const float *p) { return __ldg(p); }
    static __device__ __forceinline__ T fma(float v, T b, T a) { return fmaf(v, b, a); }
    static __device__ __forceinline__ T add(T a, T b) { return a + b; }
    static __device__ __forceinline__ void store(float *p, T v) { *p = v; }
};

// LPE lanes per output row, VW floats per lane (LPE * VW >= R); E = 32 / LPE
// rows per warp in flight.  ACC: add to C's contents (no_zero executes).
template <int LPE, int VW, bool ACC>
__global__ void __launch_bounds__(256) sym2_window_kernel(const WinParams p) {
    using V = WinVec<VW>;
    using T = typename V::T;
    constexpr int E = 32 / LPE;
    __shared__ int cp[kWinMaxRows + 1];
    __shared__ int cur[kWinMaxRows];
    __shared__ int2 items[kWinCap];
    __shared__ int rr[2];
    const int tid = threadIdx.x, nt = blockDim.x;
    if (tid == 0) {
        const int k = blockIdx.x;
        rr[0] = k == 0 ? 0 : win_lower(p, static_cast<int64_t>(k) * p.capp);
        rr[1] = k + 1 == p.nblk ? static_cast<int>(p.dim) : win_lower(p, static_cast<int64_t>(k + 1) * p.capp);
    }
    __syncthreads();
    const int r0 = rr[0], r1 = rr[1], n = r1 - r0;
    if (n <= 0) return;  // block-uniform
    const int base = p.colptr[r0];
    for (int q = tid; q <= n; q += nt) {
        cp[q] = p.colptr[r0 + q] - base;
        if (q < n) cur[q] = 0;
    }
    __syncthreads();
    // 1. column lists of the block's rows from the stream segment of rows [r0 - bw, r1)
    const int h0 = p.rowptr[max(0, r0 - p.bw)], h1 = p.rowptr[r1];
    // (four entries per thread per step: their loads are independent)
    for (int e0 = h0 + tid; e0 < h1; e0 += 4 * nt) {
        int jj[4], ii[4];
        float vv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int e = e0 + u * nt;
            const bool in = e < h1;
            jj[u] = in ? __ldg(p.c1 + e) : -1;
            ii[u] = in ? __ldg(p.c0 + e) : -1;
            vv[u] = in ? __ldg(p.vals + e) : 0.f;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int j = jj[u];
            if (j >= r0 && j < r1 && ii[u] != j) {
                const int slot = cp[j - r0] + atomicAdd(&cur[j - r0], 1);
                items[slot] = make_int2(ii[u], __float_as_int(vv[u]));
            }
        }
    }
    __syncthreads();
    // 2. every row of the block, complete, one store
    const int lane = tid & 31, g = lane / LPE, jl = lane % LPE;
    const int col = jl * VW;
    const bool act = col < p.R;
    const int colo = act ? col : 0;  // inactive lanes read column 0 (valid) and never store
    const int R = p.R;
    for (int qq = (tid >> 5) * E + g; qq < n; qq += (nt >> 5) * E) {
        const int q = r0 + qq;
        // four independent accumulators, four entries' loads in flight (a row
        // is a short dependent chain of index load -> row gather otherwise)
        T a0 = V::zero(), a1 = V::zero(), a2 = V::zero(), a3 = V::zero();
        const float *Bc = p.B + colo;
        int e = p.rowptr[q];
        const int e1 = p.rowptr[q + 1];
        for (; e + 4 <= e1; e += 4) {                    // the row part: the stored entries of row q
            const int j0 = __ldg(p.c1 + e), j1 = __ldg(p.c1 + e + 1), j2 = __ldg(p.c1 + e + 2), j3 = __ldg(p.c1 + e + 3);
            const float v0 = __ldg(p.vals + e), v1 = __ldg(p.vals + e + 1), v2 = __ldg(p.vals + e + 2),
                        v3 = __ldg(p.vals + e + 3);
            const T b0 = V::load(Bc + static_cast<int64_t>(j0) * R), b1 = V::load(Bc + static_cast<int64_t>(j1) * R);
            const T b2 = V::load(Bc + static_cast<int64_t>(j2) * R), b3 = V::load(Bc + static_cast<int64_t>(j3) * R);
            a0 = V::fma(v0, b0, a0);
            a1 = V::fma(v1, b1, a1);
            a2 = V::fma(v2, b2, a2);
            a3 = V::fma(v3, b3, a3);
        }
        for (; e < e1; ++e) a0 = V::fma(__ldg(p.vals + e), V::load(Bc + static_cast<int64_t>(__ldg(p.c1 + e)) * R), a0);
        int t = cp[qq];
        const int t1 = cp[qq + 1];
        for (; t + 4 <= t1; t += 4) {                    // the transposed part: entries (i, q), i < q
            const int2 i0 = items[t], i1 = items[t + 1], i2 = items[t + 2], i3 = items[t + 3];
            const T b0 = V::load(Bc + static_cast<int64_t>(i0.x) * R), b1 = V::load(Bc + static_cast<int64_t>(i1.x) * R);
            const T b2 = V::load(Bc + static_cast<int64_t>(i2.x) * R), b3 = V::load(Bc + static_cast<int64_t>(i3.x) * R);
            a0 = V::fma(__int_as_float(i0.y), b0, a0);
            a1 = V::fma(__int_as_float(i1.y), b1, a1);
            a2 = V::fma(__int_as_float(i2.y), b2, a2);
            a3 = V::fma(__int_as_float(i3.y), b3, a3);
        }
        for (; t < t1; ++t) {
            const int2 it = items[t];
            a0 = V::fma(__int_as_float(it.y), V::load(Bc + static_cast<int64_t>(it.x) * R), a0);
        }
        T acc = V::add(V::add(a0, a1), V::add(a2, a3));
        float *out = p.C + static_cast<int64_t>(q) * R + colo;
        if (act) {
            if (ACC) acc = V::add(acc, V::load(out));
            V::store(out, acc);
        }
    }
}

using WinFn = void (*)(WinParams);

template <int VW, bool ACC>
WinFn pick_lpe(int lpe) {
    switch (lpe) {
        case 1: return sym2_window_kernel<1, VW, ACC>;
        case 2: return sym2_window_kernel<2, VW, ACC>;
        case 4: return sym2_window_kernel<4, VW, ACC>;
        case 8: return sym2_window_kernel<8, VW, ACC>;
        case 16: return sym2_window_kernel<16, VW, ACC>;
        case 32: return sym2_window_kernel<32, VW, ACC>;
        default: return nullptr;
    }
}

int pow2ceil(int x) {
    int p = 1;
    while (p < x) p <<= 1;
    return p;
}

}  // namespace

// Plan creation, order-2 symmetric lexicographic plans: rowptr, the upper
// triangle's column pointer, the bandwidth and the largest column count
// (into *bw_dev / *maxcol_dev; the caller reads them with the statistics).
cudaError_t win_build(const Plan &p, int32_t *rowptr, int32_t *colptr, unsigned long long *bw_dev,
                      unsigned long long *maxcol_dev, cudaStream_t s) {
    const int32_t *c0 = p.coords, *c1 = p.coords + p.ld;
    cudaError_t e;
    if ((e = cudaMemsetAsync(colptr, 0, static_cast<size_t>(p.dim + 1) * 4, s)) != cudaSuccess) return e;
    if ((e = cudaMemsetAsync(bw_dev, 0, 8, s)) != cudaSuccess) return e;
    if ((e = cudaMemsetAsync(maxcol_dev, 0, 8, s)) != cudaSuccess) return e;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int blocks = sms * 8;
    win_rowptr_kernel<<<blocks, 256, 0, s>>>(c0, p.nnz, p.dim, rowptr);
    if (p.nnz > 0) win_colcount_kernel<<<blocks, 256, 0, s>>>(c0, c1, p.nnz, colptr, bw_dev);
    win_maxcol_kernel<<<blocks, 256, 0, s>>>(colptr, p.dim, maxcol_dev);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    // exclusive scan of the counts in place -> column pointer [dim + 1]
    size_t tmp = 0;
    if ((e = cub::DeviceScan::ExclusiveSum(nullptr, tmp, colptr, colptr, p.dim + 1, s)) != cudaSuccess) return e;
    void *t = nullptr;
    if ((e = cudaMallocAsync(&t, tmp, s)) != cudaSuccess) return e;
    e = cub::DeviceScan::ExclusiveSum(t, tmp, colptr, colptr, p.dim + 1, s);
    cudaFreeAsync(t, s);
    return e;
}

// Host decision from the built statistics: the partition step (0 = no window path)
int win_partition(int64_t dim, int64_t items, int64_t bw, int64_t maxcol, int *nblk) {
    const int64_t capp = kWinCap - (maxcol + kWinRowW);
    if (capp < kWinCap / 2 || dim < 1) return 0;                 // a hub column: lists would not fit
    const int64_t total = items + kWinRowW * dim;
    const int64_t nb = (total + capp - 1) / capp;
    if (nb < 1 || nb > (1 << 30)) return 0;
    if (bw > std::max<int64_t>(64, dim / nb)) return 0;          // halo larger than a block: not worth it
    *nblk = static_cast<int>(nb);
    return static_cast<int>(capp);
}

cudaError_t launch_sym2_window(const Plan &p, const float *B, int R, float *C, bool accumulate, cudaStream_t s) {
    if (p.order != 2 || p.general || !p.win_rowptr || p.win_capp <= 0) return cudaErrorNotSupported;
    const bool vec = R % 4 == 0 && (reinterpret_cast<uintptr_t>(B) % 16 == 0) && (reinterpret_cast<uintptr_t>(C) % 16 == 0);
    const int lpe = pow2ceil(vec ? R / 4 : R);
    if (lpe > 32) return cudaErrorNotSupported;
    WinFn fn = vec ? (accumulate ? pick_lpe<4, true>(lpe) : pick_lpe<4, false>(lpe))
                   : (accumulate ? pick_lpe<1, true>(lpe) : pick_lpe<1, false>(lpe));
    if (!fn) return cudaErrorNotSupported;
    WinParams wp;
    wp.c0 = p.coords;
    wp.c1 = p.coords + p.ld;
    wp.vals = p.vals;
    wp.rowptr = p.win_rowptr;
    wp.colptr = p.win_colptr;
    wp.B = B;
    wp.C = C;
    wp.dim = p.dim;
    wp.bw = static_cast<int>(p.win_bw);
    wp.capp = p.win_capp;
    wp.nblk = p.win_nblk;
    wp.R = R;
    fn<<<p.win_nblk, 256, 0, s>>>(wp);
    Plan::LaunchInfo li;
    li.grid_x = p.win_nblk;
    li.grid_y = 1;
    li.block = 256;
    li.smem = 0;
    // kernel id: 2e9 marks the windowed order-2 kernel; then vw | lpe (2 digits)
    li.kernel = 2000000000 + (vec ? 4 : 1) * 10000 + lpe * 100;
    p.record_launch(li);
    return cudaGetLastError();
}

}  // namespace systec
