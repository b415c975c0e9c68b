// mttkrp_kernel.cuh — the sm_100a symmetric sparse MTTKRP kernel template
// (SURVEY.md §8(a) a3-a6).  Instantiated per order in mttkrp_n{2,3,4,5}.cu.
//
// What one stored canonical entry e = (c_0 <= ... <= c_{n-1}; v) contributes
// (PAPER.md:859-865 for the MTTKRP, Listings 6/7 PAPER.md:685-729 for the
// symmetrised form, coef_table.cuh for the factors):
//
//     for every run-first position t:   C[c_t, r] += coef[code][t] * v * prod_{s != t} B[c_s, r]
//
// i.e. one read of the canonical entry, one gather per B
// row the entry names (common tensor access elimination),
// and one update per distinct index position (distributive grouping,
// PAPER.md:577-591), diagonals included through the coefficient table (no
// separate loop nest: this departs from Listing 7's diagonal splitting,
// PAPER.md:616-638).
//
// B200 mapping
//   * persistent grid; each warp owns a contiguous, nnz-balanced range of the
//     sorted stream (the nonzero-parallel loop with atomic output updates that
//     PAPER.md:918 names as future work);
//   * the range is consumed in chunks of CH = E*K entries that one elected lane
//     stages into shared memory with 1-D bulk async copies (TMA engine,
//     `cp.async.bulk` + mbarrier, evict-first L2 policy), in a ring of S stages;
//   * a warp is split into E = 32/LPE lane groups; group g walks entries
//     [g*K, (g+1)*K) of the chunk (K odd => the E groups hit distinct smem
//     banks); its LPE lanes spread over the rank dimension, VPL float4 (or one
//     float) per lane; B rows (rank-contiguous: the concordant B_T of
//     Listing 7) are gathered with 16-byte loads under an evict-last L2 policy;
//   * position 0: entries are sorted, so equal leading indices are contiguous;
//     the group keeps the running sum in registers (the workspace
//     transformation) and writes it only when c_0 changes;
//     at the chunk end a segmented shuffle reduction merges the groups'
//     pending sums and the last segment is carried into the next chunk;
//   * position 1 optionally accumulates the same way along runs of equal c_1;
//   * every other run-first position issues a vector `red.global.add.v4.f32`.
#pragma once
#include <cassert>
#include <cstdint>

#include "coef_table.cuh"
#include "internal.cuh"
#include "ptx.cuh"

namespace systec {

// one copy per translation unit (no relocatable device code needed)
static __constant__ CoefTable kCoef = make_coef_table();

struct KParams {
    const int32_t *coords;  // [N][ld]
    const float *vals;      // [ld]
    const float *B;         // [dim][R]
    float *C;               // [dim][R]
    int64_t ld;
    int64_t nnz;
    int64_t span;           // entries per warp (multiple of 4)
    uint32_t R;
    int K;                  // entries per lane group per chunk
    int stages;             // shared-memory ring depth
    int hints;              // 1: evict-last policy on B gathers, 0: evict-normal
    int copies;             // replicas of C the warps spread their reductions over (>= 1)
    int64_t plane;          // dim * R (floats per replica)
    int64_t dim;            // rows of B and C (bounds checks in SYSTEC_DEBUG builds)
    // work distribution: ctr != nullptr -> dynamic (warps take units of `unit`
    // consecutive entries from this zeroed counter); nullptr -> one static
    // nnz-balanced range of `span` entries per warp
    unsigned int *ctr;
    int unit;
};

using KernelFn = void (*)(KParams);

template <int VW> struct VecT;
template <> struct VecT<4> {
    using T = float4;
    static __device__ __forceinline__ T zero() { return make_float4(0.f, 0.f, 0.f, 0.f); }
    // mul2 / add2: scalar pairs by default, packed FMUL2 / FADD2 with -DSYSTEC_F32X2 (ptx.cuh)
    static __device__ __forceinline__ T mul(T a, T b) {
        T r;
        mul2(r.x, r.y, a.x, a.y, b.x, b.y);
        mul2(r.z, r.w, a.z, a.w, b.z, b.w);
        return r;
    }
    static __device__ __forceinline__ T scale(float s, T a) {
        T r;
        mul2(r.x, r.y, s, s, a.x, a.y);
        mul2(r.z, r.w, s, s, a.z, a.w);
        return r;
    }
    static __device__ __forceinline__ T add(T a, T b) {
        T r;
        add2(r.x, r.y, a.x, a.y, b.x, b.y);
        add2(r.z, r.w, a.z, a.w, b.z, b.w);
        return r;
    }
    static __device__ __forceinline__ T load(const float *p, uint64_t pol) { return ldg4_hint(p, pol); }
    static __device__ __forceinline__ void red(float *p, T v) { red_add4(p, v); }
    static __device__ __forceinline__ void red_if(float *p, T v, bool pred) { red_add4_if(p, v, pred); }
    static __device__ __forceinline__ T shfl_down(T v, int d) {
        return make_float4(__shfl_down_sync(0xffffffffu, v.x, d), __shfl_down_sync(0xffffffffu, v.y, d),
                           __shfl_down_sync(0xffffffffu, v.z, d), __shfl_down_sync(0xffffffffu, v.w, d));
    }
    static __device__ __forceinline__ T shfl(T v, int src) {
        return make_float4(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src),
                           __shfl_sync(0xffffffffu, v.z, src), __shfl_sync(0xffffffffu, v.w, src));
    }
};
// 32-byte lanes: 8 consecutive columns per lane, one 256-bit gather; the
// reduction is two red.v4 (the widest f32 vector red)
template <> struct VecT<8> {
    using T = float8;
    static __device__ __forceinline__ float4 m4(float4 a, float4 b) { return make_float4(a.x * b.x, a.y * b.y, a.z * b.z, a.w * b.w); }
    static __device__ __forceinline__ float4 s4(float s, float4 a) { return make_float4(s * a.x, s * a.y, s * a.z, s * a.w); }
    static __device__ __forceinline__ float4 a4(float4 a, float4 b) { return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w); }
    static __device__ __forceinline__ T zero() { return T{make_float4(0.f, 0.f, 0.f, 0.f), make_float4(0.f, 0.f, 0.f, 0.f)}; }
    static __device__ __forceinline__ T mul(T a, T b) { return T{m4(a.lo, b.lo), m4(a.hi, b.hi)}; }
    static __device__ __forceinline__ T scale(float s, T a) { return T{s4(s, a.lo), s4(s, a.hi)}; }
    static __device__ __forceinline__ T add(T a, T b) { return T{a4(a.lo, b.lo), a4(a.hi, b.hi)}; }
    static __device__ __forceinline__ T load(const float *p, uint64_t pol) { return ldg8_hint(p, pol); }
    static __device__ __forceinline__ void red(float *p, T v) {
        red_add4(p, v.lo);
        red_add4(p + 4, v.hi);
    }
    static __device__ __forceinline__ void red_if(float *p, T v, bool pred) {
        red_add4_if(p, v.lo, pred);
        red_add4_if(p + 4, v.hi, pred);
    }
    static __device__ __forceinline__ T shfl_down(T v, int d) {
        return T{VecT<4>::shfl_down(v.lo, d), VecT<4>::shfl_down(v.hi, d)};
    }
    static __device__ __forceinline__ T shfl(T v, int src) { return T{VecT<4>::shfl(v.lo, src), VecT<4>::shfl(v.hi, src)}; }
};
template <> struct VecT<1> {
    using T = float;
    static __device__ __forceinline__ T zero() { return 0.f; }
    static __device__ __forceinline__ T mul(T a, T b) { return a * b; }
    static __device__ __forceinline__ T scale(float s, T a) { return s * a; }
    static __device__ __forceinline__ T add(T a, T b) { return a + b; }
    static __device__ __forceinline__ T load(const float *p, uint64_t pol) { return ldg1_hint(p, pol); }
    static __device__ __forceinline__ void red(float *p, T v) { red_add1(p, v); }
    static __device__ __forceinline__ void red_if(float *p, T v, bool pred) { red_add1_if(p, v, pred); }
    static __device__ __forceinline__ T shfl_down(T v, int d) { return __shfl_down_sync(0xffffffffu, v, d); }
    static __device__ __forceinline__ T shfl(T v, int src) { return __shfl_sync(0xffffffffu, v, src); }
};

__device__ __forceinline__ uint64_t policy_evict_normal() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
    return p;
}

// base + (u32)c * stride, as one PTX mad.wide.u32
__device__ __forceinline__ char *mad_wide(int32_t c, uint32_t stride, const char *base) {
    char *r;
    asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(r) : "r"(c), "r"(stride), "l"(base));
    return r;
}

// rank offset of row c: 32x32 -> 64-bit multiply (one IMAD.WIDE.U32)
__device__ __forceinline__ uint64_t row_off(int32_t c, uint32_t R) {
    return static_cast<uint64_t>(static_cast<uint32_t>(c)) * R;
}

// ABL (ablations for the evidence table, instantiated for the c2/c5 shapes only):
//   bit 0: no shared-memory staging (indices and values read with plain loads)
//   bit 1: no position-0 run accumulation (one reduction per entry)
// RF > 0: fixed-rank build for R == RF == the rank tile (one tile, every lane
// active) and the default chunk K: the lane's columns, row stride, activity and
// the staged arrays' offsets are compile-time, which takes the per-entry
// column/bounds bookkeeping out of the loop.
template <int N, int LPE, int VPL, int VW, bool POS1, bool PF, bool NAIVE, int ABL, int RF = 0>
__device__ __forceinline__ void mttkrp_sym_body(const KParams &p) {
    using V = VecT<VW>;
    using T = typename V::T;
    constexpr int E = 32 / LPE;          // lane groups (entries in flight) per warp
    constexpr int ARR = N + 1;           // staged arrays: c_0..c_{N-1}, v
    constexpr int QS = LPE * VW;         // column stride between a lane's vectors
    constexpr int TILE = LPE * VPL * VW; // rank columns per blockIdx.y
    static_assert(RF == 0 || RF == TILE, "fixed-rank builds cover exactly one rank tile");
    constexpr bool kFull = RF > 0;
    // fixed-rank builds also fix K at the launcher's default (default_K):
    // constant smem offsets between the staged arrays
    constexpr int KF = E == 1 ? 128 : E == 2 ? 64 : E == 4 ? 33 : E == 8 ? 17 : E == 16 ? 9 : 5;
    const int K = kFull ? KF : p.K;
    const int CH = E * K;
    const int S = p.stages;
    const int WPB = blockDim.x >> 5;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane / LPE, j = lane % LPE;

    extern __shared__ __align__(128) unsigned char smem_raw[];
    int32_t *wbuf = reinterpret_cast<int32_t *>(smem_raw) + static_cast<size_t>(warp) * S * ARR * CH;
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem_raw + static_cast<size_t>(WPB) * S * ARR * CH * 4) + warp * S;

    const bool dyn = p.ctr != nullptr;
    // per-warp, per-stage chunk descriptors {base, count} (dynamic distribution)
    int32_t *meta = reinterpret_cast<int32_t *>(smem_raw + static_cast<size_t>(WPB) * S * ARR * CH * 4 +
                                                static_cast<size_t>(WPB) * S * 8) + static_cast<size_t>(warp) * S * 2;
    const int64_t gw = static_cast<int64_t>(blockIdx.x) * WPB + warp;
    int64_t begin = 0, end = 0, nch = 0;
    if (!dyn) {
        begin = gw * p.span;
        end = min(begin + p.span, p.nnz);
        if (begin >= end) return;  // warp-uniform; no block-wide barrier below
        nch = (end - begin + CH - 1) / CH;
    }

    const uint32_t R = kFull ? static_cast<uint32_t>(RF) : p.R;
    const uint32_t Rb = R * 4u;  // row stride in bytes
    const uint32_t col0 = kFull ? static_cast<uint32_t>(j * VW) : blockIdx.y * TILE + j * VW;
    // per-lane column byte offsets; inactive lanes (col >= R) read column 0 of
    // the same row (valid memory) and never write
    bool act[VPL];
    const char *Bq[VPL];
    char *Cq[VPL];
    // small outputs are spread over `copies` replicas (L2-slice spreading):
    // warp gw accumulates into replica gw % copies, summed afterwards
    char *Cbase = reinterpret_cast<char *>(p.C + static_cast<size_t>(gw % p.copies) * p.plane);
#pragma unroll
    for (int q = 0; q < VPL; ++q) {
        const uint32_t col = col0 + q * QS;
        act[q] = kFull || col < R;
        const uint32_t ofs = act[q] ? col * 4u : 0u;
        Bq[q] = reinterpret_cast<const char *>(p.B) + ofs;
        Cq[q] = Cbase + ofs;
    }
    const uint64_t pol_keep = p.hints ? policy_evict_last() : policy_evict_normal();
    const uint64_t pol_stream = policy_evict_first();
    const float *coef = kCoef.v[N - 2][0];
    constexpr float kFact = static_cast<float>(cfact(N - 1));  // (n-1)!: every coefficient of a strict entry

    if (lane == 0) {
        for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
        fence_mbar_init();
    }
    __syncwarp();

    auto issue_at = [&](int s, int64_t cb, int64_t cnt) {
        const uint32_t bytes = static_cast<uint32_t>(((cnt + 3) & ~3ll) * 4);
        int32_t *dst = wbuf + static_cast<size_t>(s) * ARR * CH;
        mbar_arrive_expect_tx(&bars[s], bytes * ARR);
#pragma unroll
        for (int a = 0; a < N; ++a) bulk_g2s(dst + a * CH, p.coords + a * p.ld + cb, bytes, &bars[s], pol_stream);
        bulk_g2s(dst + N * CH, p.vals + cb, bytes, &bars[s], pol_stream);
    };
    auto issue = [&](int64_t k) {
        const int64_t cb = begin + k * CH;
        issue_at(static_cast<int>(k % S), cb, min(static_cast<int64_t>(CH), end - cb));
    };
    // dynamic distribution: lane 0 walks units taken from the counter; a
    // stage whose descriptor base is -1 ends the warp's stream
    // (entry positions fit in int32: nnz < 2^31, include/systec.h)
    const unsigned units = dyn ? static_cast<unsigned>((p.nnz + p.unit - 1) / p.unit) : 0u;
    unsigned du = 0;
    int dnext = 0, dend = 0;  // lane 0: current unit, next chunk base, unit end
    // (requesting the following unit's id one unit ahead, to overlap the
    // atomic's round trip, measured 0.5-1 % slower on c2/c5: not done)
    auto take_unit = [&]() {
        du = atomicAdd(p.ctr + (kFull ? 0 : blockIdx.y), 1u);  // one counter per rank tile
        dnext = static_cast<int>(min(static_cast<int64_t>(du) * p.unit, p.nnz));
        dend = static_cast<int>(min(p.nnz, static_cast<int64_t>(dnext) + p.unit));  // int64: no overflow near 2^31
    };
    auto issue_dyn = [&](int64_t k) {
        const int s = static_cast<int>(k % S);
        if (du < units) {
            const int cnt = min(CH, dend - dnext);
            meta[2 * s] = dnext;
            meta[2 * s + 1] = cnt;
            issue_at(s, dnext, cnt);
            dnext += cnt;
            if (dnext >= dend) take_unit();
        } else {
            meta[2 * s] = -1;
        }
    };

    constexpr bool kStage = (ABL & 1) == 0;
    if (dyn) {
        if (lane == 0) {
            take_unit();
            for (int64_t k = 0; k < S - 1; ++k) issue_dyn(k);
        }
        __syncwarp();
    } else if (kStage && lane == 0) {
        for (int64_t k = 0; k < min(static_cast<int64_t>(S - 1), nch); ++k) issue(k);
    }

    // row address of row c for the lane's vector q: one IMAD.WIDE.U32 on the
    // lane's 64-bit base (PTX mad.wide; left to itself the compiler splits it
    // into a wide multiply, an OR of the lane offset and a 64-bit add)
    auto rowB = [&](int32_t c, int q) { return reinterpret_cast<const float *>(mad_wide(c, Rb, Bq[q])); };
    auto rowC = [&](int32_t c, int q) { return reinterpret_cast<float *>(mad_wide(c, Rb, Cq[q])); };

    // running sums: position 0 (carried across chunks) and position 1
    int cur0 = -1;
    T acc0[VPL];
    int cur1 = -1;
    bool has1 = false;
    T acc1[VPL];
#pragma unroll
    for (int q = 0; q < VPL; ++q) acc0[q] = acc1[q] = V::zero();

    for (int64_t k = 0; dyn || k < nch; ++k) {
        const int s = static_cast<int>(k % S);
        int64_t cb;
        int cnt;
        if (dyn) {
            if (lane == 0) {
                fence_proxy_async_smem();
                issue_dyn(k + S - 1);
            }
            __syncwarp();
            cb = meta[2 * s];
            if (cb < 0) break;  // warp-uniform: this warp's stream is exhausted
            cnt = meta[2 * s + 1];
            mbar_wait(&bars[s], static_cast<uint32_t>((k / S) & 1));
        } else {
            if (kStage) {
                if (lane == 0 && k + S - 1 < nch) {
                    fence_proxy_async_smem();
                    issue(k + S - 1);
                }
                mbar_wait(&bars[s], static_cast<uint32_t>((k / S) & 1));
            }
            cb = begin + k * CH;
            cnt = static_cast<int>(min(static_cast<int64_t>(CH), end - cb));
        }

        const int32_t *sc = wbuf + static_cast<size_t>(s) * ARR * CH;
        const float *sv = reinterpret_cast<const float *>(sc + N * CH);
        const int lo = g * K;
        const int hi = min(lo + K, cnt);

        // one entry's operands: indices, value, and its gathered B rows
        struct Slot {
            int32_t c[N];
            float v;
            T b[N][VPL];
        };
        auto fetch = [&](int i, Slot &x) {
            if (kStage) {
#pragma unroll
                for (int t = 0; t < N; ++t) x.c[t] = sc[t * CH + i];
                x.v = sv[i];
            } else {  // ablation: plain (cached) global loads of the stream
#pragma unroll
                for (int t = 0; t < N; ++t) x.c[t] = __ldg(p.coords + t * p.ld + cb + i);
                x.v = __ldg(p.vals + cb + i);
            }
#ifdef SYSTEC_DEBUG
#pragma unroll
            for (int t = 0; t < N; ++t) assert(x.c[t] >= 0 && x.c[t] < p.dim);
            assert(cb + i < p.nnz && i < CH);
#endif
#pragma unroll
            for (int t = NAIVE ? 1 : 0; t < N; ++t)  // the naive kernel never reads B[c_0]
#pragma unroll
                for (int q = 0; q < VPL; ++q) x.b[t][q] = V::load(rowB(x.c[t], q), pol_keep);
        };
        auto consume = [&](const Slot &x) {
            T u[N][VPL];
            // run-first flags: position t updates C iff it starts a run of equal indices
            bool first[N];
            int code = 0;
            first[0] = true;
#pragma unroll
            for (int t = 1; t < N; ++t) {
                first[t] = x.c[t] != x.c[t - 1];
                code |= (!first[t]) << (t - 1);
            }
            if (NAIVE) {  // general (non-symmetric) entry: only C[c_0] += v prod_{t>=1} B[c_t]
#pragma unroll
                for (int q = 0; q < VPL; ++q) {
                    T prod = x.b[1 % N][q];
#pragma unroll
                    for (int t = 2; t < N; ++t) prod = V::mul(prod, x.b[t][q]);
                    u[0][q] = V::scale(x.v, prod);
                }
            } else {
                // u_t = coef_t v prod_{j != t} b_j.  A strict entry (code 0) has every
                // coef = (n-1)!, folded into the scalar; a diagonal entry rescales by its
                // table row below.  P_t = s prod_{j<t} b_j, Q_t = prod_{j>t} b_j.
                const bool strict = code == 0;
                const float sc0 = strict ? x.v * kFact : x.v;
#pragma unroll
                for (int q = 0; q < VPL; ++q) {
                    T P[N];
                    P[1 % N] = V::scale(sc0, x.b[0][q]);
#pragma unroll
                    for (int t = 2; t < N; ++t) P[t] = V::mul(P[t - 1], x.b[t - 1][q]);
                    T Q = x.b[N - 1][q];
                    u[N - 1][q] = P[N - 1];
#pragma unroll
                    for (int t = N - 2; t >= 1; --t) {
                        u[t][q] = V::mul(P[t], Q);
                        Q = V::mul(Q, x.b[t][q]);
                    }
                    u[0][q] = V::scale(sc0, Q);
                }
                // diagonal entry: rescale by its coefficient row (a per-lane branch;
                // a warp vote in front of it measured 2.6 % slower on c3)
                if (!strict) {
                    const float *cf = coef + code * kMaxOrder;
#pragma unroll
                    for (int t = 0; t < N; ++t) {
                        const float f = cf[t];
#pragma unroll
                        for (int q = 0; q < VPL; ++q) u[t][q] = V::scale(f, u[t][q]);
                    }
                }
            }
            // position 0: register run accumulation; the finished run is written
            // with one (predicated) vector reduction when c_0 changes
            {
                const bool flush = (ABL & 2) || x.c[0] != cur0;
#pragma unroll
                for (int q = 0; q < VPL; ++q) {
                    V::red_if(rowC(cur0, q), acc0[q], flush && cur0 >= 0 && act[q]);
                    acc0[q] = V::add(flush ? V::zero() : acc0[q], u[0][q]);  // 0 + u == u exactly
                }
                cur0 = x.c[0];
            }
            if (NAIVE) return;
            // position 1 (POS1): the same along runs of equal c_1
            if (POS1) {
                const bool flush = x.c[1] != cur1;
                const bool take = first[1];
#pragma unroll
                for (int q = 0; q < VPL; ++q) {
                    V::red_if(rowC(cur1, q), acc1[q], flush && has1 && act[q]);
                    const T base = flush ? V::zero() : acc1[q];
                    acc1[q] = take ? V::add(base, u[1][q]) : base;
                }
                has1 = flush ? take : (has1 || take);
                cur1 = x.c[1];
            }
#pragma unroll
            for (int t = POS1 ? 2 : 1; t < N; ++t)
#pragma unroll
                for (int q = 0; q < VPL; ++q) V::red_if(rowC(x.c[t], q), u[t][q], first[t] && act[q]);
        };

        if (PF) {
            // software pipeline: the next entry's gathers are in flight while
            // this one is consumed (ping-pong slots, no register copies)
            Slot xa, xb;
            int i = lo;
            if (i < hi) fetch(i, xa);
            for (; i + 1 < hi; i += 2) {
                fetch(i + 1, xb);
                consume(xa);
                if (i + 2 < hi) fetch(i + 2, xa);
                consume(xb);
            }
            if (i < hi) consume(xa);
        } else {
            for (int i = lo; i < hi; ++i) {
                Slot x;
                fetch(i, x);
                consume(x);
            }
        }
        __syncwarp();

        if (POS1) {
#pragma unroll
            for (int q = 0; q < VPL; ++q) {
                V::red_if(rowC(cur1, q), acc1[q], has1 && act[q]);
                acc1[q] = V::zero();
            }
            has1 = false;
            cur1 = -1;
        }

        // segmented suffix reduction of the groups' pending position-0 sums over
        // maximal runs of equal keys (sorted input: keys non-decreasing in g;
        // any order stays correct because a segment stops at every key change);
        // empty tail groups carry key -1
        const int key = cur0;
        const int next_key = __shfl_down_sync(0xffffffffu, key, LPE);
        bool ends = (g == E - 1) || next_key != key;  // my segment ends within [g, g + covered)
#pragma unroll
        for (int d = 1; d < E; d <<= 1) {
            const bool o_ends = __shfl_down_sync(0xffffffffu, ends, d * LPE);
            const bool take = (g + d < E) && !ends;
#pragma unroll
            for (int q = 0; q < VPL; ++q) {
                const T o = V::shfl_down(acc0[q], d * LPE);
                if (take) acc0[q] = V::add(acc0[q], o);
            }
            if (take) ends = o_ends;
        }
        const int prev_key = __shfl_up_sync(0xffffffffu, key, LPE);
        const bool head = (g == 0) || (prev_key != key);
        const int last_key = __shfl_sync(0xffffffffu, key, (E - 1) * LPE);
        // the last segment (the one containing group E-1) starts at the highest head
        const unsigned heads = __ballot_sync(0xffffffffu, head && j == 0);
        const int hl = 31 - __clz(heads);  // lane (j == 0) of the last segment's head
        // carry the last segment when the warp's next chunk continues the stream
        bool carry;
        if (dyn) carry = meta[2 * ((k + 1) % S)] == cb + cnt;
        else carry = (k + 1 < nch);
        const bool write = head && key >= 0 && !(carry && lane - j == hl);
#pragma unroll
        for (int q = 0; q < VPL; ++q) V::red_if(rowC(key, q), acc0[q], write && act[q]);
        if (carry) {
#pragma unroll
            for (int q = 0; q < VPL; ++q) {
                const T carried = V::shfl(acc0[q], hl + j);
                acc0[q] = (g == 0) ? carried : V::zero();
            }
            cur0 = (g == 0) ? last_key : -1;
        } else {
            cur0 = -1;
#pragma unroll
            for (int q = 0; q < VPL; ++q) acc0[q] = V::zero();
        }
    }
}

template <int N, int LPE, int VPL, int VW, bool POS1, bool PF, bool NAIVE = false, int ABL = 0, int RF = 0>
__global__ void __launch_bounds__(256) mttkrp_sym_kernel(const KParams p) {
    mttkrp_sym_body<N, LPE, VPL, VW, POS1, PF, NAIVE, ABL, RF>(p);
}

// occupancy variant: ask ptxas for MINB resident 256-thread blocks per SM
// (<= 65536 / (MINB*256) registers) — for gather-latency-bound inputs.  A
// separate kernel because __launch_bounds__(256, 1) is not the same request
// as __launch_bounds__(256) (ptxas then spends registers more freely).
template <int N, int LPE, int VPL, int VW, bool POS1, int MINB, int RF = 0>
__global__ void __launch_bounds__(256, MINB) mttkrp_sym_kernel_occ(const KParams p) {
    mttkrp_sym_body<N, LPE, VPL, VW, POS1, false, false, 0, RF>(p);
}

// Sum `copies` replicas Cp[copies][plane] into C[plane] (float4 when aligned);
// accumulate != 0 adds them to C's current contents (no_zero executes).
template <int G>
__global__ void reduce_copies_kernel(const float *__restrict__ Cp, float *__restrict__ C, int64_t plane, int copies,
                                     int vec, int accumulate);

// instantiation tables, one translation unit per order (mttkrp_n{2..5}.cu)
template <int N> KernelFn pick_kernel(int vw, int lpe, int vpl, bool pos1, bool pf);
template <> KernelFn pick_kernel<2>(int vw, int lpe, int vpl, bool pos1, bool pf);
template <> KernelFn pick_kernel<3>(int vw, int lpe, int vpl, bool pos1, bool pf);
template <> KernelFn pick_kernel<4>(int vw, int lpe, int vpl, bool pos1, bool pf);
template <> KernelFn pick_kernel<5>(int vw, int lpe, int vpl, bool pos1, bool pf);
// ablation variants (abl bits above) of the c2 kernel <3,8,1,4,false,false> and c5 kernel <5,4,1,4,true,false>
KernelFn pick_ablation_kernel(int order, int abl);
// occupancy variants (more resident blocks, fewer registers): order 3 at R=32
// (<3,8,1,4,pos1>, 5 blocks/SM), orders 4 and 5 at R=16 (<n,4,1,4,pos1>, 4 blocks/SM)
KernelFn occupancy3(bool pos1);
KernelFn occupancy4(bool pos1);
KernelFn occupancy5(bool pos1);
// fixed-rank builds (R == 4*lpe, float4 lanes, one tile, no prefetch): order 3
// lpe 4/8, orders 4/5 lpe 4/8, each with pos1 on/off; occ = the occupancy
// variant of the shape that has one ((3,8), (4,4), (5,4)); nullptr if none
template <int N> KernelFn pick_full_kernel(int lpe, bool pos1, bool occ);
template <> KernelFn pick_full_kernel<3>(int lpe, bool pos1, bool occ);
template <> KernelFn pick_full_kernel<4>(int lpe, bool pos1, bool occ);
template <> KernelFn pick_full_kernel<5>(int lpe, bool pos1, bool occ);
// fixed-rank builds of the naive (expanded-tensor) kernel: lpe 4 (R = 16) / 8 (R = 32)
template <int N> KernelFn pick_full_naive_kernel(int lpe);
template <> KernelFn pick_full_naive_kernel<3>(int lpe);
template <> KernelFn pick_full_naive_kernel<4>(int lpe);
template <> KernelFn pick_full_naive_kernel<5>(int lpe);
// fixed-rank builds with 32-byte lanes (8 columns per lane, 256-bit gathers):
// order 3 at R = 32 (4 lanes per entry), orders 4/5 at R = 16 (2 lanes)
template <int N> KernelFn pick_full_v8_kernel(bool pos1);
template <> KernelFn pick_full_v8_kernel<3>(bool pos1);
template <> KernelFn pick_full_v8_kernel<4>(bool pos1);
template <> KernelFn pick_full_v8_kernel<5>(bool pos1);
// the non-symmetric (expanded-tensor) baseline: position 0 only, one float4/float per lane
template <int N> KernelFn pick_naive_kernel(int vw, int lpe, bool pf);
template <> KernelFn pick_naive_kernel<2>(int vw, int lpe, bool pf);
template <> KernelFn pick_naive_kernel<3>(int vw, int lpe, bool pf);
template <> KernelFn pick_naive_kernel<4>(int vw, int lpe, bool pf);
template <> KernelFn pick_naive_kernel<5>(int vw, int lpe, bool pf);


}  // namespace systec
