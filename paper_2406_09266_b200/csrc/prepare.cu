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
#include <algorithm>

#include <cuda_pipeline.h>

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
    // warp reductions, block totals in shared memory, then one atomic per
    // counter and block (the counters share a 128-byte line: same-line atomics
    // serialise at their L2 slice)
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
    constexpr int NS = 5 + NC;  // G, expanded, lead, pos1, maxrun, hist[NC]
    __shared__ unsigned long long part[32][NS];
    G = wsum(G);
    expanded = wsum(expanded);
    lead = wsum(lead);
    pos1 = wsum(pos1);
    maxrun = wmax(maxrun);
#pragma unroll
    for (int q = 0; q < NC; ++q) hist[q] = wsum(hist[q]);
    const int warps = (blockDim.x + 31) >> 5;
    if ((threadIdx.x & 31) == 0) {
        unsigned long long *row = part[threadIdx.x >> 5];
        row[0] = G; row[1] = expanded; row[2] = lead; row[3] = pos1; row[4] = maxrun;
#pragma unroll
        for (int q = 0; q < NC; ++q) row[5 + q] = hist[q];
    }
    __syncthreads();
    if (threadIdx.x < NS) {
        const int k = threadIdx.x;
        unsigned long long tot = 0;
        for (int w = 0; w < warps; ++w) tot = k == 4 ? (part[w][k] > tot ? part[w][k] : tot) : tot + part[w][k];
        if (tot) {
            if (k == 4) atomicMax(&st->max_lead_run, tot);
            else atomicAdd(k == 0 ? &st->G : k == 1 ? &st->expanded : k == 2 ? &st->lead_runs
                           : k == 3 ? &st->pos1_runs : &st->hist[k - 5], tot);
        }
    }
}

// ---- one-pass prepare for input that is already in storage order (the
// north_star's format: canonical tuples sorted lexicographically; tuples
// spelled in another order still qualify when their canonical forms are
// sorted).  Reads the caller's tuples once and writes the structure-of-arrays
// stream, the validation verdict, the sortedness flag and the plan statistics
// — what canonicalize + gather + stats do in three passes over packed keys.
// No keys: any order * ceil(log2 dim).  When the flag comes back "unsorted"
// the stream it wrote is discarded and the sorting path runs.
// A block stages a contiguous tile of kPrepTile tuples in shared memory with
// coalesced cp.async (16 bytes when idx is aligned; the tuples are 4N bytes apart: read per thread
// they would be strided), double-buffered; every thread then takes FOUR
// CONSECUTIVE entries: its tuples come out of shared memory as N 16-byte
// loads, an entry's predecessor is the thread's previous entry (the first one
// takes it from the tile, the tile's first from global memory), and the SoA
// stream leaves as one 16-byte store per coordinate array and one for the
// values.  Orbit sizes come from a compile-time table indexed by the equality
// pattern, the pattern histogram is kept in packed 8-bit fields.  (The first
// version took strided entries with scalar stores and recomputed factorials
// per entry: 213 instructions per entry, issue-bound at 88-94 us on c2.)
// The longest leading run is found by max_lead_run_kernel right after: a
// search per run end is bounded work only on sorted input, so that kernel
// first reads the flag.
constexpr int kPrepThreads = 256;
constexpr int kPrepU = 4;
constexpr int kPrepTile = kPrepThreads * kPrepU;

// n! / prod m_w! of an equality pattern (bit t-1 set: c_t == c_{t-1})
template <int N>
struct OrbitTable {
    unsigned v[1 << (N - 1)];
};
template <int N>
constexpr OrbitTable<N> make_orbit_table() {
    OrbitTable<N> t{};
    for (int code = 0; code < (1 << (N - 1)); ++code) {
        unsigned num = 1, den = 1;
        for (int k = 2; k <= N; ++k) num *= k;
        int run = 1;
        for (int b = 1; b < N; ++b) {
            if (code & (1 << (b - 1))) {
                ++run;
                den *= run;  // run! built up one factor at a time
            } else {
                run = 1;
            }
        }
        t.v[code] = num / den;
    }
    return t;
}
template <int N>
__device__ __forceinline__ unsigned orbit_of(int code) {
    constexpr OrbitTable<N> tab = make_orbit_table<N>();
    unsigned r = tab.v[0];
#pragma unroll
    for (int q = 1; q < (1 << (N - 1)); ++q) r = code == q ? tab.v[q] : r;  // selects on immediates: no memory
    return r;
}

template <int N, bool CANON>
__global__ void __launch_bounds__(kPrepThreads) prepare_sorted_kernel(const int32_t *__restrict__ idx,
                                                                      const float *__restrict__ vals_in, int64_t nnz,
                                                                      int64_t ld, int64_t dim,
                                                                      int32_t *__restrict__ coords,
                                                                      float *__restrict__ vals_out, DevStats *st,
                                                                      int64_t e_offset) {
    constexpr int NC = 1 << (N - 1);  // equality patterns
    constexpr int U = kPrepU;
    static_assert(U == 4, "16-byte stores of four consecutive entries");
    constexpr int HW = (NC + 7) / 8;  // 64-bit words of packed 8-bit pattern counters
    __shared__ __align__(16) int32_t tiles_s[2][kPrepTile * N];
    __shared__ bool stop;
    unsigned hist[NC];  // per-thread counts fit 32 bits (a thread sees < 2^31 / threads entries)
#pragma unroll
    for (int c = 0; c < NC; ++c) hist[c] = 0;
    unsigned long long packed[HW];
#pragma unroll
    for (int w = 0; w < HW; ++w) packed[w] = 0;
    int packed_tiles = 0;
    unsigned G = 0, expanded = 0, lead = 0, pos1 = 0;
    long long bad_at = -1;
    bool unsorted = false;
    const int tid = threadIdx.x;
    const uint32_t udim = static_cast<uint32_t>(dim);  // dim < 2^31: one unsigned compare per index
    const bool idx16 = (reinterpret_cast<uintptr_t>(idx) & 15) == 0;
    const int64_t tiles = (ld + kPrepTile - 1) / kPrepTile;
    auto canonical = [&](const int32_t *w, int32_t (&c)[N]) {  // tuple at w -> canonical c; in range?
        bool ok = true;
#pragma unroll
        for (int t = 0; t < N; ++t) {
            c[t] = w[t];
            ok &= static_cast<uint32_t>(c[t]) < udim;
        }
        if (CANON) sort_net<N>(c);
        return ok;
    };
    auto flush_packed = [&]() {
#pragma unroll
        for (int q = 0; q < NC; ++q) hist[q] += static_cast<unsigned>((packed[q / 8] >> (8 * (q % 8))) & 0xffull);
#pragma unroll
        for (int w = 0; w < HW; ++w) packed[w] = 0;
        packed_tiles = 0;
    };
    // two-stage pipeline: the next tile's tuples (4-byte cp.async into the other
    // shared buffer) are in flight while this one is consumed
    auto issue = [&](int64_t tl, int32_t *dst) {
        const int64_t base = tl * kPrepTile;
        const int64_t have = min(static_cast<int64_t>(kPrepTile), nnz - base);  // tuples of the tile (<= 0: padding only)
        const int64_t words = have > 0 ? have * N : 0;
        const int32_t *src = idx + base * N;  // 16-byte aligned when idx is (a tile is 1024 N words)
        if (idx16) {
            const int vecs = static_cast<int>(words >> 2);
#pragma unroll
            for (int k = 0; k < N; ++k) {
                const int x = tid + k * kPrepThreads;
                if (x < vecs) __pipeline_memcpy_async(dst + 4 * x, src + 4 * x, 16);
            }
            const int w = 4 * vecs + tid;  // up to three words left in a ragged last tile
            if (w < words) __pipeline_memcpy_async(dst + w, src + w, 4);
        } else {
#pragma unroll
            for (int k = 0; k < U * N; ++k) {
                const int w = tid + k * kPrepThreads;
                if (w < words) __pipeline_memcpy_async(dst + w, src + w, 4);
            }
        }
        __pipeline_commit();
    };
    int buf = 0;
    if (blockIdx.x < tiles) issue(blockIdx.x, tiles_s[0]);
    for (int64_t tl = blockIdx.x; tl < tiles; tl += gridDim.x) {
        const int64_t base = tl * kPrepTile;
        const int32_t *tile = tiles_s[buf];
        const bool more = tl + gridDim.x < tiles;
        if (more) issue(tl + gridDim.x, tiles_s[buf ^ 1]);
        const int i0 = tid * U;
        const int64_t e0 = base + i0;
        // this thread's four values (vals_in + e0 is 16-byte aligned when vals_in is; else scalar)
        float v[U];
        if (e0 + U <= nnz && (reinterpret_cast<uintptr_t>(vals_in) & 15) == 0) {
            const float4 f = *reinterpret_cast<const float4 *>(vals_in + e0);
            v[0] = f.x; v[1] = f.y; v[2] = f.z; v[3] = f.w;
        } else {
#pragma unroll
            for (int u = 0; u < U; ++u) v[u] = e0 + u < nnz ? vals_in[e0 + u] : 0.0f;
        }
        if (more) __pipeline_wait_prior(1); else __pipeline_wait_prior(0);
        // unsorted input: some block has said so — stop (what this pass wrote is discarded anyway)
        if (tid == 0) stop = *reinterpret_cast<volatile unsigned long long *>(&st->unsorted) != 0ull;
        __syncthreads();
        if (stop) {  // block-uniform
            __pipeline_wait_prior(0);
            break;
        }
        if (e0 < ld) {  // ld and e0 are multiples of 4: all four entries are inside the arrays
            int32_t out[N][U];
            int32_t q[N];
            bool qok = false;  // predecessor present and in range
            if (e0 > 0 && e0 <= nnz) qok = canonical(i0 > 0 ? tile + (i0 - 1) * N : idx + (e0 - 1) * N, q);
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int64_t e = e0 + u;
                int32_t c[N];
                bool ok = false;
                if (e < nnz) ok = canonical(tile + (i0 + u) * N, c);
#pragma unroll
                for (int t = 0; t < N; ++t) out[t][u] = ok ? c[t] : 0;  // past nnz: the padding the last chunk's bulk copies read
                if (e < nnz && !ok && bad_at < 0) bad_at = e;
                if (ok) {
                    bool new_lead = true, new_pos1 = true;
                    if (qok) {
                        bool gt = false, eq = true;  // q > c lexicographically?
#pragma unroll
                        for (int t = 0; t < N; ++t) {
                            gt |= eq & (q[t] > c[t]);
                            eq &= q[t] == c[t];
                        }
                        unsorted |= gt;
                        new_lead = q[0] != c[0];
                        new_pos1 = q[1 % N] != c[1 % N];
                    }
                    int code = 0;
#pragma unroll
                    for (int t = 1; t < N; ++t) code |= (c[t] == c[t - 1]) << (t - 1);
                    G += N - __popc(code);
                    expanded += orbit_of<N>(code);
                    const unsigned long long inc = 1ull << (8 * (code & 7));
#pragma unroll
                    for (int w = 0; w < HW; ++w) packed[w] += (code >> 3) == w ? inc : 0ull;  // no dynamic register index
                    lead += new_lead;
                    pos1 += new_pos1;
                }
#pragma unroll
                for (int t = 0; t < N; ++t) q[t] = c[t];
                qok = ok;
            }
#pragma unroll
            for (int t = 0; t < N; ++t)
                *reinterpret_cast<int4 *>(coords + t * ld + e0) = make_int4(out[t][0], out[t][1], out[t][2], out[t][3]);
            *reinterpret_cast<float4 *>(vals_out + e0) = make_float4(v[0], v[1], v[2], v[3]);
        }
        if (++packed_tiles == 63) flush_packed();  // 4 entries per tile: no 8-bit field passes 252
        // this buffer is consumed (the next round's copies may overwrite it); a disorder
        // seen in this tile is published at once
        if (__syncthreads_or(unsorted) && tid == 0) *reinterpret_cast<volatile unsigned long long *>(&st->unsorted) = 1ull;
        buf ^= 1;
    }
    flush_packed();
    if (bad_at >= 0) {
        atomicOr(&st->err, 1ull);
        atomicMin(&st->bad_entry, static_cast<unsigned long long>(bad_at + e_offset));
    }
    // block totals in shared memory, then one atomic per counter and block:
    // the counters share one 128-byte line, and same-line atomics serialise at
    // their L2 slice (one set per warp cost more than the streaming itself)
    constexpr int NS = 4 + NC;
    __shared__ unsigned long long part[kPrepThreads / 32][NS];
    auto wsum = [](unsigned long long x) {
        for (int d = 16; d; d >>= 1) x += __shfl_down_sync(0xffffffffu, x, d);
        return x;
    };
    const unsigned long long Gs = wsum(G), xs = wsum(expanded), ls = wsum(lead), ps = wsum(pos1);
    unsigned long long hs[NC];
#pragma unroll
    for (int w = 0; w < NC; ++w) hs[w] = wsum(hist[w]);
    if ((tid & 31) == 0) {
        unsigned long long *row = part[tid >> 5];
        row[0] = Gs; row[1] = xs; row[2] = ls; row[3] = ps;
#pragma unroll
        for (int w = 0; w < NC; ++w) row[4 + w] = hs[w];
    }
    __syncthreads();
    if (tid < NS) {
        unsigned long long tot = 0;
#pragma unroll
        for (int w = 0; w < kPrepThreads / 32; ++w) tot += part[w][tid];
        unsigned long long *dst = tid == 0 ? &st->G : tid == 1 ? &st->expanded : tid == 2 ? &st->lead_runs
                                  : tid == 3 ? &st->pos1_runs : &st->hist[tid - 4];
        if (tot) atomicAdd(dst, tot);
    }
}

// longest run of equal c_0 in a sorted SoA stream (c0 16-byte aligned, padded
// to a multiple of 4); returns at once when the one-pass prepare found the
// input unsorted (st->unsorted, final by stream order).  A lane holds 16
// consecutive entries, a warp a window of 512.  A run that ends in the window
// starts right after the previous run end: inside the lane, or in an earlier
// lane (an exclusive max-scan of the lanes' last ends), else before the window
// — then, and only for the window's first run end, by a galloping search
// backwards from the window's start (probes stay within twice the run's
// length) and a bisection.  One search per warp at most: with a search per
// run end the kernel was a chain of dependent loads per warp (43 us on c2).
constexpr int kRunQuads = 4;  // int4 loads per lane
__global__ void __launch_bounds__(256) max_lead_run_kernel(const int32_t *__restrict__ c0, int64_t nnz, DevStats *st) {
    if (__ldg(&st->unsorted) != 0ull) return;  // cached load: one L2 request per SM, not one per warp
    constexpr int PER = 4 * kRunQuads;
    const int lane = threadIdx.x & 31;
    const int64_t first = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * PER;  // grid covers nnz: one window per warp
    const int64_t wstart = first - static_cast<int64_t>(lane) * PER;
    unsigned long long maxrun = 0;
    if (wstart < nnz) {  // warp-uniform
        int32_t me[PER + 1];
#pragma unroll
        for (int q = 0; q < kRunQuads; ++q) {
            int4 w = make_int4(0, 0, 0, 0);
            if (first + 4 * q < nnz) w = reinterpret_cast<const int4 *>(c0 + first)[q];  // padded to a multiple of 4
            me[4 * q] = w.x; me[4 * q + 1] = w.y; me[4 * q + 2] = w.z; me[4 * q + 3] = w.w;
        }
        me[PER] = __shfl_down_sync(0xffffffffu, me[0], 1);
        if (lane == 31 && first + PER < nnz) me[PER] = c0[first + PER];
        // this lane's run ends (bit k: entry first + k ends a leading run)
        unsigned ends = 0;
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const int64_t e = first + k;
            if (e < nnz && (e == nnz - 1 || me[k + 1] != me[k])) ends |= 1u << k;
        }
        // last run end in earlier lanes of the window (-1: none)
        long long last = ends ? first + (31 - __clz(ends)) : -1;
        long long before = __shfl_up_sync(0xffffffffu, last, 1);
        if (lane == 0) before = -1;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const long long o = __shfl_up_sync(0xffffffffu, before, d);
            if (lane >= d) before = o > before ? o : before;
        }
        long long prev = before;
        while (ends) {
            const int k = __ffs(ends) - 1;
            ends &= ends - 1;
            const int64_t e = first + k;
            int64_t start;
            if (prev >= 0) {
                start = prev + 1;
            } else {  // the window's first run end: every entry from the window's start to e equals me[k]
                const int32_t val = c0[e];
                int64_t step = 1, hi2 = wstart;
                while (hi2 - step >= 0 && c0[hi2 - step] >= val) {
                    hi2 -= step;
                    step <<= 1;
                }
                int64_t lo2 = hi2 - step >= 0 ? hi2 - step + 1 : 0;  // c0[lo2 - 1] < val (or lo2 == 0); c0[hi2] == val
                while (lo2 < hi2) {
                    const int64_t mid = (lo2 + hi2) >> 1;
                    if (c0[mid] < val) lo2 = mid + 1; else hi2 = mid;
                }
                start = lo2;
            }
            const unsigned long long len = static_cast<unsigned long long>(e - start + 1);
            maxrun = len > maxrun ? len : maxrun;
            prev = e;
        }
    }
    for (int d = 16; d; d >>= 1) {
        const unsigned long long o = __shfl_down_sync(0xffffffffu, maxrun, d);
        maxrun = o > maxrun ? o : maxrun;
    }
    // one atomic per block at most, and none when the running maximum already
    // covers it (same-address atomics serialise at their L2 slice)
    __shared__ unsigned long long wmax[8];
    if (lane == 0) wmax[threadIdx.x >> 5] = maxrun;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long m = 0;
        for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) m = wmax[w] > m ? wmax[w] : m;
        if (m > *reinterpret_cast<volatile unsigned long long *>(&st->max_lead_run)) atomicMax(&st->max_lead_run, m);
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

cudaError_t launch_prepare_sorted(int order, int64_t dim, int64_t nnz, int64_t ld, const int32_t *idx,
                                  const float *vals_in, int32_t *coords, float *vals_out, DevStats *st,
                                  cudaStream_t s, bool canonicalise, int64_t e_offset) {
    if (ld == 0) return cudaSuccess;
    const int th = kPrepThreads;
    // persistent grid of exactly the resident blocks (tiles are taken round-robin: a second,
    // partial wave of blocks would leave the SMs half empty behind it), at most one block per tile
    auto resident = [&](auto kernel) {
        int dev = 0, sms = 148, per_sm = 1;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, th, 0) != cudaSuccess || per_sm < 1) per_sm = 1;
        const int64_t tiles = (ld + kPrepTile - 1) / kPrepTile;
        return static_cast<int>(std::min<int64_t>(tiles, static_cast<int64_t>(sms) * per_sm));
    };
    if (canonicalise) {
        SYSTEC_ORDER_SWITCH(order, prepare_sorted_kernel<N, true><<<resident(prepare_sorted_kernel<N, true>), th, 0, s>>>(idx, vals_in, nnz, ld, dim, coords, vals_out, st, e_offset));
    } else {
        SYSTEC_ORDER_SWITCH(order, prepare_sorted_kernel<N, false><<<resident(prepare_sorted_kernel<N, false>), th, 0, s>>>(idx, vals_in, nnz, ld, dim, coords, vals_out, st, e_offset));
    }
    // one 512-entry window per warp, uncapped grid
    if (nnz > 0) {
        const int64_t per_block = static_cast<int64_t>(th) * 4 * kRunQuads;
        max_lead_run_kernel<<<static_cast<unsigned>((nnz + per_block - 1) / per_block), th, 0, s>>>(coords, nnz, st);
    }
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
