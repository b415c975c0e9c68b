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

#include "internal.cuh"
#include "ptx.cuh"

namespace systec {

namespace {

__device__ __forceinline__ uint64_t pair_index(int32_t j, int32_t l) {  // j <= l
    return static_cast<uint64_t>(l) * (static_cast<uint64_t>(l) + 1) / 2 + static_cast<uint64_t>(j);
}

// lane groups of LPE lanes, one float4 of the rank per lane (R % 4 == 0, aligned)
template <int LPE>
__global__ void __launch_bounds__(256) ttm_sym3_kernel(const int32_t *__restrict__ coords, int64_t ld,
                                                       const float *__restrict__ vals, int64_t nnz,
                                                       const float *__restrict__ B, int R, float *__restrict__ Cp) {
    constexpr int E = 32 / LPE;
    const int lane = threadIdx.x & 31, g = lane / LPE, j = lane % LPE;
    const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    for (int64_t col = j * 4; col < R; col += LPE * 4) {
        for (int64_t e = gw * E + g; e < nnz; e += nw * E) {
            const int32_t c0 = __ldg(coords + e), c1 = __ldg(coords + ld + e), c2 = __ldg(coords + 2 * ld + e);
            const float v = __ldg(vals + e);
            // position 0 (always run-first): B[c0] into pair (c1, c2)
            float4 b = __ldg(reinterpret_cast<const float4 *>(B + static_cast<int64_t>(c0) * R + col));
            red_add4(Cp + pair_index(c1, c2) * R + col, make_float4(v * b.x, v * b.y, v * b.z, v * b.w));
            if (c1 != c0) {  // position 1: B[c1] into pair (c0, c2)
                b = __ldg(reinterpret_cast<const float4 *>(B + static_cast<int64_t>(c1) * R + col));
                red_add4(Cp + pair_index(c0, c2) * R + col, make_float4(v * b.x, v * b.y, v * b.z, v * b.w));
            }
            if (c2 != c1) {  // position 2: B[c2] into pair (c0, c1)
                b = __ldg(reinterpret_cast<const float4 *>(B + static_cast<int64_t>(c2) * R + col));
                red_add4(Cp + pair_index(c0, c1) * R + col, make_float4(v * b.x, v * b.y, v * b.z, v * b.w));
            }
        }
    }
}

// scalar fallback: any R, any alignment
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

// naive TTM over a GENERAL order-3 plan (e.g. the expanded tensor): every
// entry (p0, p1, p2; v) adds v B[p0, :] to the FULL output C[p1][p2][:]
__global__ void ttm_general_kernel(const int32_t *__restrict__ coords, int64_t ld, const float *__restrict__ vals,
                                   int64_t nnz, const float *__restrict__ B, int R, int64_t dim, float *__restrict__ C,
                                   int vec) {
    const int64_t per = vec ? R / 4 : R;
    const int64_t total = nnz * per;
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t e = q / per;
        const int r = static_cast<int>(q % per);
        const int32_t p0 = coords[e], p1 = coords[ld + e], p2 = coords[2 * ld + e];
        const float v = vals[e];
        float *c = C + (static_cast<int64_t>(p1) * dim + p2) * R;
        const float *b = B + static_cast<int64_t>(p0) * R;
        if (vec) {
            const float4 x = __ldg(reinterpret_cast<const float4 *>(b) + r);
            red_add4(c + 4 * r, make_float4(v * x.x, v * x.y, v * x.z, v * x.w));
        } else {
            atomicAdd(c + r, v * b[r]);
        }
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
        ttm_general_kernel<<<blocks, 256, 0, s>>>(p.coords, p.ld, p.vals, p.nnz, B, R, p.dim, Cp, vec ? 1 : 0);
        return cudaGetLastError();
    }
    if (vec) {
        const int vecs = R / 4;
        int lpe = 1;
        while (lpe < vecs && lpe < 32) lpe <<= 1;
        switch (lpe) {
            case 1: ttm_sym3_kernel<1><<<blocks, 256, 0, s>>>(p.coords, p.ld, p.vals, p.nnz, B, R, Cp); break;
            case 2: ttm_sym3_kernel<2><<<blocks, 256, 0, s>>>(p.coords, p.ld, p.vals, p.nnz, B, R, Cp); break;
            case 4: ttm_sym3_kernel<4><<<blocks, 256, 0, s>>>(p.coords, p.ld, p.vals, p.nnz, B, R, Cp); break;
            case 8: ttm_sym3_kernel<8><<<blocks, 256, 0, s>>>(p.coords, p.ld, p.vals, p.nnz, B, R, Cp); break;
            case 16: ttm_sym3_kernel<16><<<blocks, 256, 0, s>>>(p.coords, p.ld, p.vals, p.nnz, B, R, Cp); break;
            default: ttm_sym3_kernel<32><<<blocks, 256, 0, s>>>(p.coords, p.ld, p.vals, p.nnz, B, R, Cp); break;
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
