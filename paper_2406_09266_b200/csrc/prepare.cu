// prepare.cu — device-side validation, canonicalisation, lexicographic sort and
// structure-of-arrays gather of the stored COO entries.
//
// Paper basis: a fully symmetric tensor is determined by its canonical triangle
// (Def. Symmetry, Def. Canonical), so every
// input tuple is replaced by its ascending sort; the symmetrised kernel then
// walks only canonical coordinates ("if p_1 <= ... <= p_n").
// The concordant, sorted traversal order corresponds to building the CSF /
// concordising step of PAPER.md:482-503.  The paper excludes this
// rearrangement from its timings; so do we (plan creation).
#include <cub/device/device_radix_sort.cuh>

#include "internal.cuh"

namespace systec {

namespace {

template <int N>
__device__ __forceinline__ void sort_net(int32_t (&c)[N]) {
    // odd-even transposition network, fully unrolled (N <= 5)
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

template <int N>
__device__ __forceinline__ unsigned long long pack_key(const int32_t (&c)[N], int bits) {
    unsigned long long k = 0;
#pragma unroll
    for (int t = 0; t < N; ++t) k = (k << bits) | static_cast<unsigned long long>(static_cast<uint32_t>(c[t]));
    return k;
}

template <int N, bool CANON>
__device__ __forceinline__ bool load_canonical(const int32_t *idx, int64_t e, int64_t dim, int32_t (&c)[N]) {
    bool ok = true;
#pragma unroll
    for (int t = 0; t < N; ++t) {
        c[t] = idx[e * N + t];
        ok &= (c[t] >= 0) & (static_cast<int64_t>(c[t]) < dim);
    }
    if (CANON) sort_net<N>(c);  // a general (non-symmetric) tensor keeps its tuples as given
    return ok;
}

template <int N, bool CANON>
__global__ void canonicalize_kernel(const int32_t *__restrict__ idx, int64_t nnz, int64_t dim, int bits,
                                    unsigned long long *__restrict__ keys, uint32_t *__restrict__ perm,
                                    DevStats *st, int64_t e_offset) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz;
         e += (int64_t)gridDim.x * blockDim.x) {
        int32_t c[N];
        const bool ok = load_canonical<N, CANON>(idx, e, dim, c);
        if (!ok) {
            atomicOr(&st->err, 1ull);
            atomicMin(&st->bad_entry, static_cast<unsigned long long>(e + e_offset));
            keys[e] = 0;
            perm[e] = static_cast<uint32_t>(e);
            continue;
        }
        const unsigned long long k = pack_key<N>(c, bits);
        keys[e] = k;
        perm[e] = static_cast<uint32_t>(e);
        if (e > 0) {
            int32_t q[N];
            if (load_canonical<N, CANON>(idx, e - 1, dim, q) && pack_key<N>(q, bits) > k) st->unsorted = 1ull;
        }
    }
}

template <int N>
__global__ void gather_kernel(int64_t nnz, int64_t ld, int bits, const unsigned long long *__restrict__ keys,
                              const uint32_t *__restrict__ perm, const float *__restrict__ vals_in,
                              int32_t *__restrict__ coords, float *__restrict__ vals_out) {
    const unsigned long long mask = (bits >= 64) ? ~0ull : ((1ull << bits) - 1ull);
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ld;
         e += (int64_t)gridDim.x * blockDim.x) {
        if (e < nnz) {
            unsigned long long k = keys[e];
#pragma unroll
            for (int t = N - 1; t >= 0; --t) {
                coords[t * ld + e] = static_cast<int32_t>(k & mask);
                k >>= bits;
            }
            vals_out[e] = vals_in[perm ? perm[e] : e];
        } else {  // padding read by the bulk copies of the last chunk; never used
#pragma unroll
            for (int t = 0; t < N; ++t) coords[t * ld + e] = 0;
            vals_out[e] = 0.0f;
        }
    }
}

// chunk form for the pipelined host path: n entries, no permutation, no padding
template <int N>
__global__ void gather_range_kernel(int64_t n, int64_t ld, int bits, const unsigned long long *__restrict__ keys,
                                    const float *__restrict__ vals_in, int32_t *__restrict__ coords,
                                    float *__restrict__ vals_out) {
    const unsigned long long mask = (bits >= 64) ? ~0ull : ((1ull << bits) - 1ull);
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        unsigned long long k = keys[e];
#pragma unroll
        for (int t = N - 1; t >= 0; --t) {
            coords[t * ld + e] = static_cast<int32_t>(k & mask);
            k >>= bits;
        }
        vals_out[e] = vals_in[e];
    }
}

// ---- wide plans: order * ceil(log2 dim) > 64, the canonical tuple does not
// fit one 64-bit key.  Nothing is packed: validation compares neighbouring
// tuples directly, the sort is an LSD radix sort over words of `cpw`
// coordinates each (last word first, every pass stable, carrying only the
// permutation), and the gather re-reads the caller's tuples through it.

template <int N, bool CANON>
__global__ void validate_wide_kernel(const int32_t *__restrict__ idx, int64_t nnz, int64_t dim,
                                     uint32_t *__restrict__ perm, DevStats *st, int64_t e_offset) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz;
         e += (int64_t)gridDim.x * blockDim.x) {
        int32_t c[N];
        perm[e] = static_cast<uint32_t>(e);
        if (!load_canonical<N, CANON>(idx, e, dim, c)) {
            atomicOr(&st->err, 1ull);
            atomicMin(&st->bad_entry, static_cast<unsigned long long>(e + e_offset));
            continue;
        }
        if (e > 0) {
            int32_t q[N];
            if (load_canonical<N, CANON>(idx, e - 1, dim, q)) {
                int cmp = 0;  // sign of q - c in lexicographic order
#pragma unroll
                for (int t = 0; t < N; ++t)
                    if (cmp == 0) cmp = (q[t] > c[t]) - (q[t] < c[t]);
                if (cmp > 0) st->unsorted = 1ull;
            }
        }
    }
}

// keys[e] = coordinates [first, first + count) of the canonical tuple of entry perm[e]
template <int N, bool CANON>
__global__ void word_keys_kernel(const int32_t *__restrict__ idx, int64_t nnz, int64_t dim, int bits, int first,
                                 int count, const uint32_t *__restrict__ perm,
                                 unsigned long long *__restrict__ keys) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz;
         e += (int64_t)gridDim.x * blockDim.x) {
        int32_t c[N];
        load_canonical<N, CANON>(idx, perm[e], dim, c);
        unsigned long long k = 0;
#pragma unroll
        for (int t = 0; t < N; ++t)
            if (t >= first && t < first + count)
                k = (k << bits) | static_cast<unsigned long long>(static_cast<uint32_t>(c[t]));
        keys[e] = k;
    }
}

template <int N, bool CANON>
__global__ void gather_wide_kernel(int64_t nnz, int64_t span, int64_t ld, int64_t dim,
                                   const int32_t *__restrict__ idx, const uint32_t *__restrict__ perm,
                                   const float *__restrict__ vals_in, int32_t *__restrict__ coords,
                                   float *__restrict__ vals_out) {
    // span = ld for a whole plan (entries past nnz are padding), = nnz for one chunk of the host pipeline
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < span;
         e += (int64_t)gridDim.x * blockDim.x) {
        if (e < nnz) {
            const int64_t src = perm ? static_cast<int64_t>(perm[e]) : e;
            int32_t c[N];
            load_canonical<N, CANON>(idx, src, dim, c);
#pragma unroll
            for (int t = 0; t < N; ++t) coords[t * ld + e] = c[t];
            vals_out[e] = vals_in[src];
        } else {  // padding (see gather_kernel)
#pragma unroll
            for (int t = 0; t < N; ++t) coords[t * ld + e] = 0;
            vals_out[e] = 0.0f;
        }
    }
}

// banded stream order (systec_plan_opts.band_shift): the band number of each
// prepared entry, c_{N-1} >> band_shift, with its position
template <int N>
__global__ void band_keys_kernel(int64_t nnz, int64_t ld, const int32_t *__restrict__ coords, int band_shift,
                                 uint16_t *__restrict__ band, uint32_t *__restrict__ perm) {
    const int32_t *cl = coords + static_cast<int64_t>(N - 1) * ld;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz;
         e += (int64_t)gridDim.x * blockDim.x) {
        band[e] = static_cast<uint16_t>(static_cast<uint32_t>(cl[e]) >> band_shift);
        perm[e] = static_cast<uint32_t>(e);
    }
}

// out[t][e] = in[t][perm[e]], vals likewise; the padding tail is zeroed
template <int N>
__global__ void permute_kernel(int64_t nnz, int64_t ld, const uint32_t *__restrict__ perm,
                               const int32_t *__restrict__ cin, const float *__restrict__ vin,
                               int32_t *__restrict__ cout, float *__restrict__ vout) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ld;
         e += (int64_t)gridDim.x * blockDim.x) {
        if (e < nnz) {
            const int64_t src = perm[e];
#pragma unroll
            for (int t = 0; t < N; ++t) cout[t * ld + e] = cin[t * ld + src];
            vout[e] = vin[src];
        } else {
#pragma unroll
            for (int t = 0; t < N; ++t) cout[t * ld + e] = 0;
            vout[e] = 0.0f;
        }
    }
}

__device__ __forceinline__ long long dfact(int k) {
    long long f = 1;
    for (int i = 2; i <= k; ++i) f *= i;
    return f;
}

template <int N>
__global__ void stats_kernel(int64_t nnz, int64_t ld, const int32_t *__restrict__ coords, int band_shift,
                             DevStats *st) {
    constexpr int NC = 1 << (N - 1);  // equality patterns
    unsigned long long hist[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) hist[c] = 0;
    unsigned long long G = 0, expanded = 0, lead = 0, pos1 = 0, maxrun = 0;
    const int32_t *c0 = coords;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz;
         e += (int64_t)gridDim.x * blockDim.x) {
        int32_t c[N];
#pragma unroll
        for (int t = 0; t < N; ++t) c[t] = coords[t * ld + e];
        int code = 0, distinct = 1, run = 1;
        long long denom = 1;
#pragma unroll
        for (int t = 1; t < N; ++t) {
            if (c[t] == c[t - 1]) {
                code |= 1 << (t - 1);
                ++run;
            } else {
                ++distinct;
                denom *= dfact(run);
                run = 1;
            }
        }
        denom *= dfact(run);
        G += distinct;
        expanded += static_cast<unsigned long long>(dfact(N) / denom);
#pragma unroll
        for (int q = 0; q < NC; ++q) hist[q] += (code == q);
        if (e == 0 || c0[e - 1] != c[0]) ++lead;
        if (N >= 2 && (e == 0 || coords[ld + e - 1] != c[1])) ++pos1;
        if (e == nnz - 1 || c0[e + 1] != c[0]) {  // end of a leading run: its start by binary search
            // over (band, c_0), the leading part of the sort key
            const int32_t *cl = coords + static_cast<int64_t>(N - 1) * ld;
            auto lead_key = [&](int64_t x) {
                const uint32_t b = band_shift >= 0 ? static_cast<uint32_t>(cl[x]) >> band_shift : 0u;
                return (static_cast<unsigned long long>(b) << 32) | static_cast<uint32_t>(c0[x]);
            };
            const unsigned long long me = lead_key(e);
            int64_t lo = 0, hi = e;
            while (lo < hi) {
                const int64_t mid = (lo + hi) >> 1;
                if (lead_key(mid) < me) lo = mid + 1; else hi = mid;
            }
            const unsigned long long len = static_cast<unsigned long long>(e - lo + 1);
            maxrun = len > maxrun ? len : maxrun;
        }
    }
    // warp reductions, then one atomic per warp and counter
    auto wsum = [](unsigned long long v) {
        for (int d = 16; d; d >>= 1) v += __shfl_down_sync(0xffffffffu, v, d);
        return v;
    };
    auto wmax = [](unsigned long long v) {
        for (int d = 16; d; d >>= 1) {
            const unsigned long long o = __shfl_down_sync(0xffffffffu, v, d);
            v = o > v ? o : v;
        }
        return v;
    };
    G = wsum(G);
    expanded = wsum(expanded);
    lead = wsum(lead);
    pos1 = wsum(pos1);
    maxrun = wmax(maxrun);
#pragma unroll
    for (int q = 0; q < NC; ++q) hist[q] = wsum(hist[q]);
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(&st->G, G);
        atomicAdd(&st->expanded, expanded);
        atomicAdd(&st->lead_runs, lead);
        atomicAdd(&st->pos1_runs, pos1);
        if (maxrun) atomicMax(&st->max_lead_run, maxrun);
#pragma unroll
        for (int q = 0; q < NC; ++q)
            if (hist[q]) atomicAdd(&st->hist[q], hist[q]);
    }
}

int grid_for(int64_t n, int threads) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t want = (n + threads - 1) / threads;
    const int64_t cap = static_cast<int64_t>(sms) * 16;
    return static_cast<int>(want < 1 ? 1 : (want > cap ? cap : want));
}

}  // namespace

#define SYSTEC_ORDER_SWITCH(order, ...)          \
    switch (order) {                             \
        case 2: { constexpr int N = 2; __VA_ARGS__; } break; \
        case 3: { constexpr int N = 3; __VA_ARGS__; } break; \
        case 4: { constexpr int N = 4; __VA_ARGS__; } break; \
        case 5: { constexpr int N = 5; __VA_ARGS__; } break; \
        default: return cudaErrorInvalidValue;   \
    }

cudaError_t launch_canonicalize(int order, int64_t dim, int64_t nnz, int bits, const int32_t *idx,
                                unsigned long long *keys, uint32_t *perm, DevStats *st, cudaStream_t s,
                                bool canonicalise, int64_t e_offset) {
    if (nnz == 0) return cudaSuccess;
    const int th = 256;
    if (canonicalise) {
        SYSTEC_ORDER_SWITCH(order, canonicalize_kernel<N, true><<<grid_for(nnz, th), th, 0, s>>>(idx, nnz, dim, bits, keys, perm, st, e_offset));
    } else {
        SYSTEC_ORDER_SWITCH(order, canonicalize_kernel<N, false><<<grid_for(nnz, th), th, 0, s>>>(idx, nnz, dim, bits, keys, perm, st, e_offset));
    }
    return cudaGetLastError();
}

cudaError_t sort_keys(int64_t nnz, int end_bit, unsigned long long *keys_in, unsigned long long *keys_out,
                      uint32_t *perm_in, uint32_t *perm_out, cudaStream_t s) {
    size_t temp = 0;
    cudaError_t e = cub::DeviceRadixSort::SortPairs(nullptr, temp, keys_in, keys_out, perm_in, perm_out,
                                                    static_cast<int>(nnz), 0, end_bit, s);
    if (e != cudaSuccess) return e;
    void *tmp = nullptr;
    e = cudaMallocAsync(&tmp, temp ? temp : 16, s);
    if (e != cudaSuccess) return e;
    e = cub::DeviceRadixSort::SortPairs(tmp, temp, keys_in, keys_out, perm_in, perm_out,
                                        static_cast<int>(nnz), 0, end_bit, s);
    cudaError_t f = cudaFreeAsync(tmp, s);
    return e != cudaSuccess ? e : f;
}

cudaError_t launch_gather(int order, int64_t nnz, int64_t ld, int bits, const unsigned long long *keys,
                          const uint32_t *perm, const float *vals_in, int32_t *coords, float *vals_out,
                          cudaStream_t s) {
    if (ld == 0) return cudaSuccess;
    const int th = 256;
    SYSTEC_ORDER_SWITCH(order, gather_kernel<N><<<grid_for(ld, th), th, 0, s>>>(nnz, ld, bits, keys, perm, vals_in, coords, vals_out));
    return cudaGetLastError();
}

cudaError_t launch_validate_wide(int order, int64_t dim, int64_t nnz, const int32_t *idx, uint32_t *perm,
                                 DevStats *st, cudaStream_t s, bool canonicalise, int64_t e_offset) {
    if (nnz == 0) return cudaSuccess;
    const int th = 256;
    if (canonicalise) {
        SYSTEC_ORDER_SWITCH(order, validate_wide_kernel<N, true><<<grid_for(nnz, th), th, 0, s>>>(idx, nnz, dim, perm, st, e_offset));
    } else {
        SYSTEC_ORDER_SWITCH(order, validate_wide_kernel<N, false><<<grid_for(nnz, th), th, 0, s>>>(idx, nnz, dim, perm, st, e_offset));
    }
    return cudaGetLastError();
}

// Lexicographic sort of the canonical tuples for wide plans: perm (identity on
// entry) becomes the sorting permutation.  keys/keys2 [nnz] 64-bit and perm2
// [nnz] are scratch; the result is in *perm_out (perm or perm2).
cudaError_t sort_wide(int order, int64_t dim, int64_t nnz, int bits, const int32_t *idx, unsigned long long *keys,
                      unsigned long long *keys2, uint32_t *perm, uint32_t *perm2, uint32_t **perm_out,
                      cudaStream_t s, bool canonicalise) {
    const int cpw = 64 / bits;                    // coordinates per 64-bit word (bits <= 31: at least 2)
    const int words = (order + cpw - 1) / cpw;
    const int th = 256;
    uint32_t *in = perm, *out = perm2;
    for (int w = words - 1; w >= 0; --w) {
        const int first = w * cpw, count = order - first < cpw ? order - first : cpw;
        if (canonicalise) {
            SYSTEC_ORDER_SWITCH(order, word_keys_kernel<N, true><<<grid_for(nnz, th), th, 0, s>>>(idx, nnz, dim, bits, first, count, in, keys));
        } else {
            SYSTEC_ORDER_SWITCH(order, word_keys_kernel<N, false><<<grid_for(nnz, th), th, 0, s>>>(idx, nnz, dim, bits, first, count, in, keys));
        }
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        if ((e = sort_keys(nnz, bits * count, keys, keys2, in, out, s)) != cudaSuccess) return e;
        uint32_t *t = in; in = out; out = t;
    }
    *perm_out = in;
    return cudaSuccess;
}

cudaError_t launch_gather_wide(int order, int64_t nnz, int64_t span, int64_t ld, int64_t dim, const int32_t *idx,
                               const uint32_t *perm, const float *vals_in, int32_t *coords, float *vals_out,
                               cudaStream_t s, bool canonicalise) {
    if (span == 0) return cudaSuccess;
    const int th = 256;
    if (canonicalise) {
        SYSTEC_ORDER_SWITCH(order, gather_wide_kernel<N, true><<<grid_for(span, th), th, 0, s>>>(nnz, span, ld, dim, idx, perm, vals_in, coords, vals_out));
    } else {
        SYSTEC_ORDER_SWITCH(order, gather_wide_kernel<N, false><<<grid_for(span, th), th, 0, s>>>(nnz, span, ld, dim, idx, perm, vals_in, coords, vals_out));
    }
    return cudaGetLastError();
}

cudaError_t launch_band_keys(int order, int64_t nnz, int64_t ld, const int32_t *coords, int band_shift,
                             uint16_t *band, uint32_t *perm, cudaStream_t s) {
    if (nnz == 0) return cudaSuccess;
    const int th = 256;
    SYSTEC_ORDER_SWITCH(order, band_keys_kernel<N><<<grid_for(nnz, th), th, 0, s>>>(nnz, ld, coords, band_shift, band, perm));
    return cudaGetLastError();
}

// stable (LSD radix) sort of (band, position) pairs on the band's bits only
cudaError_t sort_band_keys(int64_t nnz, int band_bits, uint16_t *keys_in, uint16_t *keys_out, uint32_t *perm_in,
                           uint32_t *perm_out, cudaStream_t s) {
    size_t temp = 0;
    cudaError_t e = cub::DeviceRadixSort::SortPairs(nullptr, temp, keys_in, keys_out, perm_in, perm_out,
                                                    static_cast<int>(nnz), 0, band_bits, s);
    if (e != cudaSuccess) return e;
    void *tmp = nullptr;
    e = cudaMallocAsync(&tmp, temp ? temp : 16, s);
    if (e != cudaSuccess) return e;
    e = cub::DeviceRadixSort::SortPairs(tmp, temp, keys_in, keys_out, perm_in, perm_out, static_cast<int>(nnz), 0,
                                        band_bits, s);
    cudaError_t f = cudaFreeAsync(tmp, s);
    return e != cudaSuccess ? e : f;
}

cudaError_t launch_permute(int order, int64_t nnz, int64_t ld, const uint32_t *perm, const int32_t *cin,
                           const float *vin, int32_t *cout, float *vout, cudaStream_t s) {
    if (ld == 0) return cudaSuccess;
    const int th = 256;
    SYSTEC_ORDER_SWITCH(order, permute_kernel<N><<<grid_for(ld, th), th, 0, s>>>(nnz, ld, perm, cin, vin, cout, vout));
    return cudaGetLastError();
}

cudaError_t launch_gather_range(int order, int64_t n, int64_t ld, int bits, const unsigned long long *keys,
                                const float *vals_in, int32_t *coords, float *vals_out, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const int th = 256;
    SYSTEC_ORDER_SWITCH(order, gather_range_kernel<N><<<grid_for(n, th), th, 0, s>>>(n, ld, bits, keys, vals_in, coords, vals_out));
    return cudaGetLastError();
}

cudaError_t launch_stats(int order, int64_t nnz, int64_t ld, const int32_t *coords, int band_shift, DevStats *st,
                         cudaStream_t s) {
    if (nnz == 0) return cudaSuccess;
    const int th = 256;
    SYSTEC_ORDER_SWITCH(order, stats_kernel<N><<<grid_for(nnz, th), th, 0, s>>>(nnz, ld, coords, band_shift, st));
    return cudaGetLastError();
}

}  // namespace systec
