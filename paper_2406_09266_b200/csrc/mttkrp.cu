// mttkrp.cu — the sm_100a symmetric sparse MTTKRP kernel.
//
// What one stored canonical entry e = (c_0 <= ... <= c_{n-1}; v) contributes
// (PAPER.md:859-865 for the MTTKRP, Listing 6/7 PAPER.md:685-729 for the
// symmetrised form, coef_table.cuh for the factors):
//
//     for every run-first position t:   C[c_t, r] += coef[code][t] * v * prod_{s != t} B[c_s, r]
//
// i.e. one read of the canonical entry, one gather of each
// distinct B row (common tensor access elimination), and one
// update per distinct index position (distributive grouping),
// diagonals included through the coefficient table (no separate loop nest:
// this is where we depart from Listing 7's diagonal splitting).
//
// B200 mapping
//   * persistent grid; each warp owns a contiguous, nnz-balanced range of the
//     sorted stream (the nonzero-parallel loop with atomic output updates that
//     PAPER.md:918 names as future work);
//   * the range is consumed in chunks of CH = E*K entries that one elected lane
//     stages into shared memory with 1-D bulk async copies (TMA engine,
//     `cp.async.bulk` + mbarrier, evict-first L2 policy), double-buffered;
//   * a warp is split into E = 32/LPE lane groups; group g walks entries
//     [g*K, (g+1)*K) of the chunk, its LPE lanes spread across the rank
//     dimension with one float4 (or float) per lane — B rows (rank-contiguous,
//     the concordant B_T of Listing 7) are gathered with 16-byte loads under an
//     evict-last L2 policy so B stays L2-resident;
//   * position 0: entries are sorted, so equal leading indices are contiguous;
//     the group keeps the running sum in registers (the workspace
//     transformation) and writes it only when c_0 changes;
//     at the chunk end a segmented shuffle reduction merges the groups'
//     pending sums and the last segment is carried into the next chunk;
//   * position 1 optionally accumulates the same way along runs of equal c_1;
//   * every other run-first position issues a vector `red.global.add.v4.f32`.
#include <algorithm>

#include "coef_table.cuh"
#include "internal.cuh"
#include "ptx.cuh"

namespace systec {

__constant__ CoefTable kCoef = make_coef_table();

namespace {

template <int VW> struct VecT;
template <> struct VecT<4> {
    using T = float4;
    static __device__ __forceinline__ T zero() { return make_float4(0.f, 0.f, 0.f, 0.f); }
    static __device__ __forceinline__ T splat(float a) { return make_float4(a, a, a, a); }
    static __device__ __forceinline__ T mul(T a, T b) { return make_float4(a.x * b.x, a.y * b.y, a.z * b.z, a.w * b.w); }
    static __device__ __forceinline__ T scale(float s, T a) { return make_float4(s * a.x, s * a.y, s * a.z, s * a.w); }
    static __device__ __forceinline__ T add(T a, T b) { return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w); }
    static __device__ __forceinline__ T load(const float *p, uint64_t pol, bool hint) {
        return hint ? ldg4_hint(p, pol) : ldg4(p);
    }
    static __device__ __forceinline__ void red(float *p, T v) { red_add4(p, v); }
    static __device__ __forceinline__ T shfl_down(T v, int d) {
        return make_float4(__shfl_down_sync(0xffffffffu, v.x, d), __shfl_down_sync(0xffffffffu, v.y, d),
                           __shfl_down_sync(0xffffffffu, v.z, d), __shfl_down_sync(0xffffffffu, v.w, d));
    }
    static __device__ __forceinline__ T shfl(T v, int src) {
        return make_float4(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src),
                           __shfl_sync(0xffffffffu, v.z, src), __shfl_sync(0xffffffffu, v.w, src));
    }
};
template <> struct VecT<1> {
    using T = float;
    static __device__ __forceinline__ T zero() { return 0.f; }
    static __device__ __forceinline__ T splat(float a) { return a; }
    static __device__ __forceinline__ T mul(T a, T b) { return a * b; }
    static __device__ __forceinline__ T scale(float s, T a) { return s * a; }
    static __device__ __forceinline__ T add(T a, T b) { return a + b; }
    static __device__ __forceinline__ T load(const float *p, uint64_t pol, bool hint) {
        return hint ? ldg1_hint(p, pol) : ldg1(p);
    }
    static __device__ __forceinline__ void red(float *p, T v) { red_add1(p, v); }
    static __device__ __forceinline__ T shfl_down(T v, int d) { return __shfl_down_sync(0xffffffffu, v, d); }
    static __device__ __forceinline__ T shfl(T v, int src) { return __shfl_sync(0xffffffffu, v, src); }
};

struct KParams {
    const int32_t *coords;  // [N][ld]
    const float *vals;      // [ld]
    const float *B;         // [dim][R]
    float *C;               // [dim][R]
    int64_t ld;
    int64_t nnz;
    int64_t span;           // entries per warp (multiple of 4)
    int R;
    int K;                  // entries per lane group per chunk
    int stages;             // shared-memory ring depth
    int hints;              // L2 cache-policy hints on/off
};

template <int N, int LPE, int VW, bool POS1>
__global__ void __launch_bounds__(256) mttkrp_sym_kernel(const KParams p) {
    using V = VecT<VW>;
    using T = typename V::T;
    constexpr int E = 32 / LPE;   // lane groups (entries in flight) per warp
    constexpr int ARR = N + 1;    // staged arrays: c_0..c_{N-1}, v
    const int K = p.K;
    const int CH = E * K;
    const int S = p.stages;
    const int WPB = blockDim.x >> 5;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane / LPE, j = lane % LPE;

    extern __shared__ __align__(128) unsigned char smem_raw[];
    int32_t *wbuf = reinterpret_cast<int32_t *>(smem_raw) + static_cast<size_t>(warp) * S * ARR * CH;
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem_raw + static_cast<size_t>(WPB) * S * ARR * CH * 4) + warp * S;

    const int64_t gw = static_cast<int64_t>(blockIdx.x) * WPB + warp;
    const int64_t begin = gw * p.span;
    const int64_t end = min(begin + p.span, p.nnz);
    if (begin >= end) return;  // warp-uniform; no block-wide barrier below
    const int64_t nch = (end - begin + CH - 1) / CH;

    const int col = blockIdx.y * (LPE * VW) + j * VW;
    const bool active = col < p.R;
    const int64_t R = p.R;
    const float *Bc = p.B + col;
    float *Cc = p.C + col;
    const bool hint = p.hints != 0;
    const uint64_t pol_keep = policy_evict_last();
    const uint64_t pol_stream = policy_evict_first();
    const float *coef = kCoef.v[N - 2][0];

    if (lane == 0) {
        for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
        fence_mbar_init();
    }
    __syncwarp();

    auto issue = [&](int64_t k) {
        const int s = static_cast<int>(k % S);
        const int64_t cb = begin + k * CH;
        const int64_t cnt = min(static_cast<int64_t>(CH), end - cb);
        const uint32_t bytes = static_cast<uint32_t>(((cnt + 3) & ~3ll) * 4);
        int32_t *dst = wbuf + static_cast<size_t>(s) * ARR * CH;
        mbar_arrive_expect_tx(&bars[s], bytes * ARR);
#pragma unroll
        for (int a = 0; a < N; ++a) bulk_g2s(dst + a * CH, p.coords + a * p.ld + cb, bytes, &bars[s], pol_stream);
        bulk_g2s(dst + N * CH, p.vals + cb, bytes, &bars[s], pol_stream);
    };

    if (lane == 0)
        for (int64_t k = 0; k < min(static_cast<int64_t>(S - 1), nch); ++k) issue(k);

    // running sums: position 0 (carried across chunks) and position 1
    int cur0 = -1;
    T acc0 = V::zero();
    int cur1 = -1;
    bool has1 = false;
    T acc1 = V::zero();

    for (int64_t k = 0; k < nch; ++k) {
        if (lane == 0 && k + S - 1 < nch) {
            fence_proxy_async_smem();
            issue(k + S - 1);
        }
        const int s = static_cast<int>(k % S);
        mbar_wait(&bars[s], static_cast<uint32_t>((k / S) & 1));

        const int32_t *sc = wbuf + static_cast<size_t>(s) * ARR * CH;
        const float *sv = reinterpret_cast<const float *>(sc + N * CH);
        const int64_t cb = begin + k * CH;
        const int cnt = static_cast<int>(min(static_cast<int64_t>(CH), end - cb));
        const int lo = g * K;
        const int hi = min(lo + K, cnt);

        for (int i = lo; i < hi; ++i) {
            int c[N];
#pragma unroll
            for (int t = 0; t < N; ++t) c[t] = sc[t * CH + i];
            const float v = sv[i];
            int code = 0;
#pragma unroll
            for (int t = 0; t + 1 < N; ++t) code |= (c[t] == c[t + 1]) << t;
            const float *cf = coef + code * kMaxOrder;

            T b[N];
            if (active) {
                b[0] = V::load(Bc + c[0] * R, pol_keep, hint);
#pragma unroll
                for (int t = 1; t < N; ++t)
                    b[t] = (c[t] == c[t - 1]) ? b[t - 1] : V::load(Bc + c[t] * R, pol_keep, hint);
            } else {
#pragma unroll
                for (int t = 0; t < N; ++t) b[t] = V::zero();
            }
            // prefix / suffix products: u_t = (coef_t v) prod_{s<t} b_s prod_{s>t} b_s
            T pre[N];
            pre[0] = V::splat(1.f);
#pragma unroll
            for (int t = 1; t < N; ++t) pre[t] = (t == 1) ? b[0] : V::mul(pre[t - 1], b[t - 1]);
            T u[N];
            T suf = V::splat(1.f);
#pragma unroll
            for (int t = N - 1; t >= 0; --t) {
                const T prod = (t == N - 1) ? pre[t] : (t == 0 ? suf : V::mul(pre[t], suf));
                u[t] = V::scale(cf[t] * v, prod);
                if (t > 0) suf = (t == N - 1) ? b[t] : V::mul(suf, b[t]);
            }

            // position 0: register run accumulation
            if (c[0] != cur0) {
                if (cur0 >= 0 && active) V::red(Cc + cur0 * R, acc0);
                cur0 = c[0];
                acc0 = V::zero();
            }
            acc0 = V::add(acc0, u[0]);
            // position 1
            if (POS1) {
                if (c[1] != cur1) {
                    if (has1 && active) V::red(Cc + cur1 * R, acc1);
                    cur1 = c[1];
                    acc1 = V::zero();
                    has1 = false;
                }
                if (cf[1] != 0.f) {
                    acc1 = V::add(acc1, u[1]);
                    has1 = true;
                }
            }
#pragma unroll
            for (int t = POS1 ? 2 : 1; t < N; ++t)
                if (cf[t] != 0.f && active) V::red(Cc + c[t] * R, u[t]);
        }
        __syncwarp();

        if (POS1) {
            if (has1 && active) V::red(Cc + cur1 * R, acc1);
            has1 = false;
            cur1 = -1;
            acc1 = V::zero();
        }

        // segmented reduction of the groups' pending position-0 sums
        // (keys are non-decreasing in g; empty groups carry key -1 at the tail)
        const int key = cur0;
#pragma unroll
        for (int d = 1; d < E; d <<= 1) {
            const T o = V::shfl_down(acc0, d * LPE);
            const int ok = __shfl_down_sync(0xffffffffu, key, d * LPE);
            if (g + d < E && ok == key) acc0 = V::add(acc0, o);
        }
        const int prev_key = __shfl_up_sync(0xffffffffu, key, LPE);
        const bool head = (g == 0) || (prev_key != key);
        const int last_key = __shfl_sync(0xffffffffu, key, (E - 1) * LPE);
        const bool carry = (k + 1 < nch);  // chunk was full: next chunk continues the stream
        if (head && key >= 0 && active && !(carry && key == last_key)) V::red(Cc + key * R, acc0);
        if (carry) {
            const unsigned heads = __ballot_sync(0xffffffffu, head && j == 0 && key == last_key);
            const int hl = __ffs(heads) - 1;  // lane of the last segment's head (j == 0)
            const T carried = V::shfl(acc0, hl + j);
            cur0 = (g == 0) ? last_key : -1;
            acc0 = (g == 0) ? carried : V::zero();
        } else {
            cur0 = -1;
            acc0 = V::zero();
        }
    }
}

using KernelFn = void (*)(KParams);

template <int N, int LPE, int VW>
KernelFn pick_pos1(bool pos1) {
    return pos1 ? mttkrp_sym_kernel<N, LPE, VW, true> : mttkrp_sym_kernel<N, LPE, VW, false>;
}
template <int N, int VW>
KernelFn pick_lpe(int lpe, bool pos1) {
    switch (lpe) {
        case 1: return pick_pos1<N, 1, VW>(pos1);
        case 2: return pick_pos1<N, 2, VW>(pos1);
        case 4: return pick_pos1<N, 4, VW>(pos1);
        case 8: return pick_pos1<N, 8, VW>(pos1);
        case 16: return pick_pos1<N, 16, VW>(pos1);
        default: return pick_pos1<N, 32, VW>(pos1);
    }
}
template <int N>
KernelFn pick_vw(int vw, int lpe, bool pos1) {
    return vw == 4 ? pick_lpe<N, 4>(lpe, pos1) : pick_lpe<N, 1>(lpe, pos1);
}
KernelFn pick(int order, int vw, int lpe, bool pos1) {
    switch (order) {
        case 2: return pick_vw<2>(vw, lpe, pos1);
        case 3: return pick_vw<3>(vw, lpe, pos1);
        case 4: return pick_vw<4>(vw, lpe, pos1);
        case 5: return pick_vw<5>(vw, lpe, pos1);
        default: return nullptr;
    }
}

int pow2ceil(int x) {
    int p = 1;
    while (p < x) p <<= 1;
    return p;
}

}  // namespace

cudaError_t launch_mttkrp(Plan &p, const float *B, int R, float *C, const systec_exec_opts &o, cudaStream_t s) {
    cudaError_t e;
    if (!o.no_zero) {
        e = cudaMemsetAsync(C, 0, static_cast<size_t>(p.dim) * R * sizeof(float), s);
        if (e != cudaSuccess) return e;
    }
    if (p.nnz == 0) return cudaSuccess;

    const bool aligned = (reinterpret_cast<uintptr_t>(B) % 16 == 0) && (reinterpret_cast<uintptr_t>(C) % 16 == 0);
    const int vw = (R % 4 == 0 && aligned && !o.force_scalar) ? 4 : 1;
    const int lanes_needed = (R + vw - 1) / vw;
    const int lpe = std::min(32, pow2ceil(lanes_needed));
    const int E = 32 / lpe;
    const int tiles = (R + lpe * vw - 1) / (lpe * vw);
    // K: lane groups read smem word g*K+i; K = 33 (or 17) keeps the E groups on
    // distinct banks; CH = E*K stays a multiple of 4 (16-byte bulk copies).
    int K = (E >= 4) ? (p.order >= 4 ? 17 : 33) : 32;
    if (E >= 4 && (E * K) % 4 != 0) K = 32;
    if (o.reserved[0] > 0) K = o.reserved[0];  // tuning override: entries per group per chunk
    const int stages = o.reserved[1] > 0 ? o.reserved[1] : 2;
    if ((E * K) % 4 != 0) return cudaErrorInvalidValue;

    bool pos1 = false;
    if (o.pos1_accumulate > 0) pos1 = true;
    else if (o.pos1_accumulate == 0 && p.stats.pos1_runs > 0)
        pos1 = (static_cast<double>(p.nnz) / static_cast<double>(p.stats.pos1_runs)) >= 1.5;

    KernelFn fn = pick(p.order, vw, lpe, pos1);
    if (!fn) return cudaErrorInvalidValue;
    int wpb = o.warps_per_block > 0 ? o.warps_per_block : 8;
    auto smem_for = [&](int w) {
        return static_cast<size_t>(w) * stages * (p.order + 1) * (E * K) * 4 + static_cast<size_t>(w) * stages * 8;
    };
    const size_t smem_cap = 200 * 1024;
    while (wpb > 1 && smem_for(wpb) > smem_cap) wpb >>= 1;  // keep the staging ring within shared memory
    if (smem_for(wpb) > smem_cap) return cudaErrorInvalidValue;
    const int threads = wpb * 32;
    if (threads > 256) return cudaErrorInvalidValue;
    const size_t smem = smem_for(wpb);
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 148, occ = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, threads, smem);
    if (e != cudaSuccess) return e;
    if (occ < 1) occ = 1;
    if (o.blocks_per_sm > 0) occ = std::min(occ, static_cast<int>(o.blocks_per_sm));
    const int64_t total_warps = static_cast<int64_t>(sms) * occ * wpb;
    int64_t span = (p.nnz + total_warps - 1) / total_warps;
    span = std::max<int64_t>(4, (span + 3) & ~3ll);
    const int64_t warps_used = (p.nnz + span - 1) / span;
    const int64_t blocks = (warps_used + wpb - 1) / wpb;

    KParams kp;
    kp.coords = p.coords;
    kp.vals = p.vals;
    kp.B = B;
    kp.C = C;
    kp.ld = p.ld;
    kp.nnz = p.nnz;
    kp.span = span;
    kp.R = R;
    kp.K = K;
    kp.stages = stages;
    kp.hints = o.l2_hints >= 0 ? 1 : 0;
    dim3 grid(static_cast<unsigned>(blocks), static_cast<unsigned>(tiles));
    fn<<<grid, threads, smem, s>>>(kp);
    p.last_grid_x = static_cast<int>(blocks);
    p.last_grid_y = tiles;
    p.last_block = threads;
    p.last_smem = static_cast<int>(smem);
    p.last_kernel = (p.order * 1000) + vw * 100 + lpe * 2 + (pos1 ? 1 : 0);
    return cudaGetLastError();
}

}  // namespace systec
