// ttm.cu — symmetric tensor-times-matrix with visible output symmetry
// (the paper's TTM, Listings 1-3
// PAPER.md:262-325):
//
//     C[i, j, l] = sum_k A[k, j, l] * B[k, i]        A fully symmetric, order 3
//
// C inherits the symmetry C[i,j,l] = C[i,l,j] (visible output symmetry,
// PAPER.md:217-232), so only its canonical half j <= l is computed, stored
// packed as Cp[pair(j,l)][i] (rank-contiguous rows, pair(j,l) = l(l+1)/2 + j);
// replication to the full tensor is a separate kernel (the paper excludes it
// from its timings; the output-restriction transform is
// PAPER.md:459-480).
//
// What a stored canonical entry (c0 <= c1 <= c2; v) contributes: every distinct
// permutation (p0, p1, p2) of its indices adds v B[p0, :] to C[:, p1, p2]; in
// the canonical half exactly one permutation per DISTINCT leading value p0
// survives (the other two indices sorted), so for each run-first position u:
//     Cp[pair(remaining two, sorted)][:] += v * B[c_u, :]
// with no multiplicity factor.
#include <algorithm>
#include <type_traits>

#include "internal.cuh"
#include "ptx.cuh"

namespace systec {

namespace {

__device__ __forceinline__ uint64_t pair_index(int32_t j, int32_t l) {  // j <= l
    return static_cast<uint64_t>(l) * (static_cast<uint64_t>(l) + 1) / 2 + static_cast<uint64_t>(j);
}

// Lane groups of LPE lanes, one float4 of the rank per lane (R % 4 == 0,
// aligned); every group walks a CONTIGUOUS range of the lexicographically
// sorted stream, so entries with equal (c0, c1) are consecutive and the
// position-2 update (target pair (c0, c1)) accumulates in registers along the
// run and is written with one vector reduction per run (the workspace
// transformation); positions 0 and 1 reduce per entry.
template <int LPE>
__global__ void __launch_bounds__(256) ttm_sym3_kernel(const int32_t *__restrict__ coords, int64_t ld,
                                                       const float *__restrict__ vals, int64_t nnz,
                                                       const float *__restrict__ B, int R, float *__restrict__ Cp,
                                                       int64_t span) {
    constexpr int E = 32 / LPE;
    const int lane = threadIdx.x & 31, g = lane / LPE, j = lane % LPE;
    const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t grp = gw * E + g;
    const int64_t begin = grp * span, end = min(begin + span, nnz);
    struct Ent {
        int32_t c0, c1, c2;
        float v;
    };
    auto load = [&](int64_t e) {
        Ent x;
        x.c0 = __ldg(coords + e);
        x.c1 = __ldg(coords + ld + e);
        x.c2 = __ldg(coords + 2 * ld + e);
        x.v = __ldg(vals + e);
        return x;
    };
    for (int64_t col = j * 4; col < R; col += LPE * 4) {
        auto rows = [&](const Ent &x, float4 (&b)[3]) {
            b[0] = __ldg(reinterpret_cast<const float4 *>(B + static_cast<int64_t>(x.c0) * R + col));
            b[1] = __ldg(reinterpret_cast<const float4 *>(B + static_cast<int64_t>(x.c1) * R + col));
            b[2] = __ldg(reinterpret_cast<const float4 *>(B + static_cast<int64_t>(x.c2) * R + col));
        };
        int32_t k0 = -1, k1 = -1;  // key (c0, c1) of the pending position-2 sum
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        // software pipeline: indices two entries ahead, B rows one entry ahead
        Ent cur{}, nxt{};
        float4 bc[3], bn[3];
        if (begin < end) {
            cur = load(begin);
            rows(cur, bc);
        }
        if (begin + 1 < end) nxt = load(begin + 1);
        for (int64_t e = begin; e < end; ++e) {
            Ent nn{};
            if (e + 2 < end) nn = load(e + 2);
            if (e + 1 < end) rows(nxt, bn);
            const Ent x = cur;
            const float v = x.v;
            // position 0 (always run-first): B[c0] into pair (c1, c2)
            red_add4(Cp + pair_index(x.c1, x.c2) * R + col, make_float4(v * bc[0].x, v * bc[0].y, v * bc[0].z, v * bc[0].w));
            if (x.c1 != x.c0)  // position 1: B[c1] into pair (c0, c2)
                red_add4(Cp + pair_index(x.c0, x.c2) * R + col,
                         make_float4(v * bc[1].x, v * bc[1].y, v * bc[1].z, v * bc[1].w));
            // position 2: B[c2] into pair (c0, c1), accumulated along the (c0, c1) run
            if (x.c0 != k0 || x.c1 != k1) {
                if (k0 >= 0) red_add4(Cp + pair_index(k0, k1) * R + col, acc);
                acc = make_float4(0.f, 0.f, 0.f, 0.f);
                k0 = x.c0;
                k1 = x.c1;
            }
            if (x.c2 != x.c1) {
                acc.x = fmaf(v, bc[2].x, acc.x);
                acc.y = fmaf(v, bc[2].y, acc.y);
                acc.z = fmaf(v, bc[2].z, acc.z);
                acc.w = fmaf(v, bc[2].w, acc.w);
            }
            cur = nxt;
            nxt = nn;
#pragma unroll
            for (int t = 0; t < 3; ++t) bc[t] = bn[t];
        }
        if (k0 >= 0) red_add4(Cp + pair_index(k0, k1) * R + col, acc);
    }
}

__global__ void ttm_sym3_scalar_kernel(const int32_t *__restrict__ coords, int64_t ld, const float *__restrict__ vals,
                                       int64_t nnz, const float *__restrict__ B, int R, float *__restrict__ Cp) {
    const int64_t total = nnz * R;
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t e = q / R;
        const int r = static_cast<int>(q % R);
        const int32_t c0 = coords[e], c1 = coords[ld + e], c2 = coords[2 * ld + e];
        const float v = vals[e];
        atomicAdd(Cp + pair_index(c1, c2) * R + r, v * B[static_cast<int64_t>(c0) * R + r]);
        if (c1 != c0) atomicAdd(Cp + pair_index(c0, c2) * R + r, v * B[static_cast<int64_t>(c1) * R + r]);
        if (c2 != c1) atomicAdd(Cp + pair_index(c0, c1) * R + r, v * B[static_cast<int64_t>(c2) * R + r]);
    }
}

// Naive TTM over a GENERAL order-3 plan (e.g. the expanded tensor), contracting
// the LAST mode — the one innermost in the sorted stream, so the loop order is
// concordant for the naive kernel too: every entry (p0, p1, p2; v) adds
// v B[p2, :] to the full output row C[p0][p1][:], accumulated in registers
// along the run of equal (p0, p1) and written once per run.  (For the expansion
// of a symmetric tensor this is the same C as contracting mode 0.)  Lane groups
// of LPE lanes, VW floats per lane, contiguous entry ranges.
template <int LPE, int VW>
__global__ void __launch_bounds__(256) ttm_general_kernel(const int32_t *__restrict__ coords, int64_t ld,
                                                          const float *__restrict__ vals, int64_t nnz,
                                                          const float *__restrict__ B, int R, int64_t dim,
                                                          float *__restrict__ C, int64_t span) {
    using T = typename std::conditional<VW == 4, float4, float>::type;
    constexpr int E = 32 / LPE;
    const int lane = threadIdx.x & 31, g = lane / LPE, j = lane % LPE;
    const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t grp = gw * E + g;
    const int64_t begin = grp * span, end = min(begin + span, nnz);
    struct Ent {
        int32_t p0, p1, p2;
        float v;
    };
    auto load = [&](int64_t e) {
        Ent x;
        x.p0 = __ldg(coords + e);
        x.p1 = __ldg(coords + ld + e);
        x.p2 = __ldg(coords + 2 * ld + e);
        x.v = __ldg(vals + e);
        return x;
    };
    for (int64_t col = j * VW; col < R; col += LPE * VW) {
        auto row = [&](const Ent &x) -> T {
            return __ldg(reinterpret_cast<const T *>(B + static_cast<int64_t>(x.p2) * R + col));
        };
        int32_t k0 = -1, k1 = -1;
        float acc[VW];
#pragma unroll
        for (int u = 0; u < VW; ++u) acc[u] = 0.f;
        auto flush = [&]() {
            float *c = C + (static_cast<int64_t>(k0) * dim + k1) * R + col;
            if constexpr (VW == 4) red_add4(c, make_float4(acc[0], acc[1], acc[2], acc[3]));
            else atomicAdd(c, acc[0]);
        };
        // software pipeline: indices two entries ahead, the B row one entry ahead
        Ent cur{}, nxt{};
        T bc{}, bn{};
        if (begin < end) {
            cur = load(begin);
            bc = row(cur);
        }
        if (begin + 1 < end) nxt = load(begin + 1);
        for (int64_t e = begin; e < end; ++e) {
            Ent nn{};
            if (e + 2 < end) nn = load(e + 2);
            if (e + 1 < end) bn = row(nxt);
            if (cur.p0 != k0 || cur.p1 != k1) {
                if (k0 >= 0) flush();
#pragma unroll
                for (int u = 0; u < VW; ++u) acc[u] = 0.f;
                k0 = cur.p0;
                k1 = cur.p1;
            }
            if constexpr (VW == 4) {
                acc[0] = fmaf(cur.v, bc.x, acc[0]);
                acc[1] = fmaf(cur.v, bc.y, acc[1]);
                acc[2] = fmaf(cur.v, bc.z, acc[2]);
                acc[3] = fmaf(cur.v, bc.w, acc[3]);
            } else {
                acc[0] = fmaf(cur.v, bc, acc[0]);
            }
            cur = nxt;
            nxt = nn;
            bc = bn;
        }
        if (k0 >= 0) flush();
    }
}

// C[j][l][i] = Cp[pair(min, max)][i]  (full output, rank innermost)
__global__ void ttm_unpack_kernel(const float *__restrict__ Cp, int64_t dim, int R, float *__restrict__ C) {
    const int64_t total = dim * dim * R;
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
        const int r = static_cast<int>(q % R);
        const int64_t jl = q / R;
        const int32_t j = static_cast<int32_t>(jl / dim), l = static_cast<int32_t>(jl % dim);
        C[q] = Cp[pair_index(min(j, l), max(j, l)) * R + r];
    }
}

int sms_of() {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms;
}

}  // namespace

int64_t ttm_packed_rows(int64_t dim) { return dim * (dim + 1) / 2; }

cudaError_t launch_ttm(const Plan &p, const float *B, int R, float *Cp, cudaStream_t s) {
    const size_t bytes = static_cast<size_t>(p.general ? p.dim * p.dim : ttm_packed_rows(p.dim)) * R * 4;
    cudaError_t e = cudaMemsetAsync(Cp, 0, bytes, s);
    if (e != cudaSuccess || p.nnz == 0) return e;
    const bool vec = R % 4 == 0 && reinterpret_cast<uintptr_t>(B) % 16 == 0 && reinterpret_cast<uintptr_t>(Cp) % 16 == 0;
    const int blocks = sms_of() * 8;
    if (p.general) {
        const int vw = vec ? 4 : 1;
        const int vecs = (R + vw - 1) / vw;
        int lpe = 1;
        while (lpe < vecs && lpe < 32) lpe <<= 1;
        const int64_t groups = static_cast<int64_t>(blocks) * 8 * (32 / lpe);
        const int64_t span = std::max<int64_t>(1, (p.nnz + groups - 1) / groups);
#define SYSTEC_TTM_GEN(L)                                                                                      \
    (vec ? ttm_general_kernel<L, 4><<<blocks, 256, 0, s>>>(p.coords, p.ld, p.vals, p.nnz, B, R, p.dim, Cp, span) \
         : ttm_general_kernel<L, 1><<<blocks, 256, 0, s>>>(p.coords, p.ld, p.vals, p.nnz, B, R, p.dim, Cp, span))
        switch (lpe) {
            case 1: SYSTEC_TTM_GEN(1); break;
            case 2: SYSTEC_TTM_GEN(2); break;
            case 4: SYSTEC_TTM_GEN(4); break;
            case 8: SYSTEC_TTM_GEN(8); break;
            case 16: SYSTEC_TTM_GEN(16); break;
            default: SYSTEC_TTM_GEN(32); break;
        }
#undef SYSTEC_TTM_GEN
        return cudaGetLastError();
    }
    if (vec) {
        const int vecs = R / 4;
        int lpe = 1;
        while (lpe < vecs && lpe < 32) lpe <<= 1;
        const int64_t groups = static_cast<int64_t>(blocks) * 8 * (32 / lpe);
        const int64_t span = std::max<int64_t>(1, (p.nnz + groups - 1) / groups);
        switch (lpe) {
            case 1: ttm_sym3_kernel<1><<<blocks, 256, 0, s>>>(p.coords, p.ld, p.vals, p.nnz, B, R, Cp, span); break;
            case 2: ttm_sym3_kernel<2><<<blocks, 256, 0, s>>>(p.coords, p.ld, p.vals, p.nnz, B, R, Cp, span); break;
            case 4: ttm_sym3_kernel<4><<<blocks, 256, 0, s>>>(p.coords, p.ld, p.vals, p.nnz, B, R, Cp, span); break;
            case 8: ttm_sym3_kernel<8><<<blocks, 256, 0, s>>>(p.coords, p.ld, p.vals, p.nnz, B, R, Cp, span); break;
            case 16: ttm_sym3_kernel<16><<<blocks, 256, 0, s>>>(p.coords, p.ld, p.vals, p.nnz, B, R, Cp, span); break;
            default: ttm_sym3_kernel<32><<<blocks, 256, 0, s>>>(p.coords, p.ld, p.vals, p.nnz, B, R, Cp, span); break;
        }
    } else {
        ttm_sym3_scalar_kernel<<<blocks, 256, 0, s>>>(p.coords, p.ld, p.vals, p.nnz, B, R, Cp);
    }
    return cudaGetLastError();
}

cudaError_t launch_ttm_unpack(int64_t dim, int R, const float *Cp, float *C, cudaStream_t s) {
    const int64_t total = dim * dim * R;
    const int blocks = static_cast<int>(std::min<int64_t>((total + 255) / 256, static_cast<int64_t>(sms_of()) * 16));
    ttm_unpack_kernel<<<std::max(blocks, 1), 256, 0, s>>>(Cp, dim, R, C);
    return cudaGetLastError();
}

}  // namespace systec
