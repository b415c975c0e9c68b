// mttkrp_tma.cu — EXPERIMENT: the order-3, R%32==0 MTTKRP kernel with the B-row
// gathers done by the TMA engine (`cp.async.bulk.tensor.2d ... tile::gather4`,
// SASS UTMALDG.2D.GATHER4): each warp step gathers the 12 rows of its 4 entries
// with three 4-row TMA gathers into a shared-memory ring D steps deep, so the
// gathers in flight cost no registers and no per-lane load instructions.
// Position 0 (and 1 with POS1) accumulate along runs like the main kernel;
// pending sums are flushed at every chunk end (no cross-group merge).
#include <cuda.h>

#include <algorithm>

#include "internal.cuh"
#include "ptx.cuh"

namespace systec {

namespace {

struct alignas(64) TmaParams {
    CUtensorMap tmB;         // B as a 2-D tensor {R, dim}, box {32, 1}
    const int32_t *coords;   // [3][ld]
    const float *vals;
    float *C;
    int64_t ld, nnz, span;
    uint32_t R;
    int K, stages, copies;
    int64_t plane;
};

__device__ __forceinline__ void gather4(uint32_t dst, const CUtensorMap *tm, int col, int r0, int r1, int r2, int r3,
                                        uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
        "l"(tm), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(bar))
        : "memory");
}

template <bool POS1, int D>
__global__ void __launch_bounds__(256) mttkrp3_tma_kernel(const __grid_constant__ TmaParams P) {
    constexpr int N = 3, LPE = 8, E = 4, ARR = 4, ROWS = E * N;
    const int K = P.K, CH = E * K, S = P.stages;
    const int WPB = blockDim.x >> 5;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane / LPE, j = lane % LPE;

    extern __shared__ __align__(128) unsigned char smem_raw[];
    const size_t stream_bytes = static_cast<size_t>(WPB) * S * ARR * CH * 4;
    int32_t *wbuf = reinterpret_cast<int32_t *>(smem_raw) + static_cast<size_t>(warp) * S * ARR * CH;
    const size_t ring_off = (stream_bytes + 127) & ~size_t(127);
    float *gring = reinterpret_cast<float *>(smem_raw + ring_off) + static_cast<size_t>(warp) * D * ROWS * 32;
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem_raw + ring_off + static_cast<size_t>(WPB) * D * ROWS * 128) +
                     static_cast<size_t>(warp) * (S + D);
    uint64_t *gbars = bars + S;

    const int64_t gw = static_cast<int64_t>(blockIdx.x) * WPB + warp;
    const int64_t begin = gw * P.span;
    const int64_t end = min(begin + P.span, P.nnz);
    if (begin >= end) return;
    const int64_t nch = (end - begin + CH - 1) / CH;

    const uint32_t R = P.R, Rb = R * 4u;
    const int col0 = blockIdx.y * 32;
    char *Cbase = reinterpret_cast<char *>(P.C + static_cast<size_t>(gw % P.copies) * P.plane) + (col0 + j * 4) * 4;
    auto rowC = [&](int32_t c) { return reinterpret_cast<float *>(Cbase + static_cast<uint64_t>(static_cast<uint32_t>(c)) * Rb); };
    const uint64_t pol_stream = policy_evict_first();

    if (lane == 0) {
        for (int s = 0; s < S + D; ++s) mbar_init(&bars[s], 1);
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
        for (int a = 0; a < N; ++a) bulk_g2s(dst + a * CH, P.coords + a * P.ld + cb, bytes, &bars[s], pol_stream);
        bulk_g2s(dst + N * CH, P.vals + cb, bytes, &bars[s], pol_stream);
    };
    if (lane == 0)
        for (int64_t k = 0; k < min(static_cast<int64_t>(S - 1), nch); ++k) issue(k);

    int cur0 = -1, cur1 = -1;
    bool has1 = false;
    float4 acc0 = make_float4(0, 0, 0, 0), acc1 = make_float4(0, 0, 0, 0);
    uint64_t u = 0;  // global step counter: slot u % D, parity (u / D) & 1

    for (int64_t k = 0; k < nch; ++k) {
        const int s = static_cast<int>(k % S);
        if (lane == 0 && k + S - 1 < nch) {
            fence_proxy_async_smem();
            issue(k + S - 1);
        }
        mbar_wait(&bars[s], static_cast<uint32_t>((k / S) & 1));
        const int32_t *sc = wbuf + static_cast<size_t>(s) * ARR * CH;
        const float *sv = reinterpret_cast<const float *>(sc + N * CH);
        const int64_t cb = begin + k * CH;
        const int cnt = static_cast<int>(min(static_cast<int64_t>(CH), end - cb));
        const int steps = min(K, cnt);

        auto issue_gather = [&](int st, uint64_t uu) {  // rows of step st for all 4 groups
            const int slot = static_cast<int>(uu % D);
            int r[ROWS];
#pragma unroll
            for (int gg = 0; gg < E; ++gg) {
                const int i = gg * K + st;
#pragma unroll
                for (int t = 0; t < N; ++t) r[gg * N + t] = (i < cnt) ? sc[t * CH + i] : 0;
            }
            float *dst = gring + static_cast<size_t>(slot) * ROWS * 32;
            mbar_arrive_expect_tx(&gbars[slot], ROWS * 128);
#pragma unroll
            for (int q = 0; q < ROWS / 4; ++q)
                gather4(smem_u32(dst + q * 4 * 32), &P.tmB, col0, r[4 * q], r[4 * q + 1], r[4 * q + 2], r[4 * q + 3],
                        &gbars[slot]);
        };
        if (lane == 0)
            for (int d = 0; d < D && d < steps; ++d) issue_gather(d, u + d);

        for (int st = 0; st < steps; ++st, ++u) {
            const int slot = static_cast<int>(u % D);
            mbar_wait(&gbars[slot], static_cast<uint32_t>((u / D) & 1));
            const int i = g * K + st;
            const bool valid = i < cnt;
            const float *row = gring + static_cast<size_t>(slot) * ROWS * 32;
            int32_t c[N];
            float4 b[N];
#pragma unroll
            for (int t = 0; t < N; ++t) {
                c[t] = valid ? sc[t * CH + i] : -2;
                b[t] = *reinterpret_cast<const float4 *>(row + (g * N + t) * 32 + j * 4);
            }
            const float v = valid ? sv[i] : 0.f;
            __syncwarp();
            if (lane == 0 && st + D < steps) {
                fence_proxy_async_smem();
                issue_gather(st + D, u + D);
            }
            if (valid) {
                const bool f1 = c[1] != c[0], f2 = c[2] != c[1];
                const int code = (!f1) | ((!f2) << 1);
                // coefficients of n = 3 (coef_table.cuh): 0 -> [2,2,2], 1 -> [2,0,1], 2 -> [1,2,0], 3 -> [1,0,0]
                const float k0 = (code & 2) ? 1.f : 2.f;
                const float k1 = f1 ? ((code & 2) ? 2.f : 2.f) : 0.f;
                const float k2 = f2 ? ((code & 1) ? 1.f : 2.f) : 0.f;
                const float4 p12 = make_float4(b[1].x * b[2].x, b[1].y * b[2].y, b[1].z * b[2].z, b[1].w * b[2].w);
                const float4 p02 = make_float4(b[0].x * b[2].x, b[0].y * b[2].y, b[0].z * b[2].z, b[0].w * b[2].w);
                const float4 p01 = make_float4(b[0].x * b[1].x, b[0].y * b[1].y, b[0].z * b[1].z, b[0].w * b[1].w);
                const float s0 = k0 * v, s1 = k1 * v, s2 = k2 * v;
                const float4 u0 = make_float4(s0 * p12.x, s0 * p12.y, s0 * p12.z, s0 * p12.w);
                const float4 u1 = make_float4(s1 * p02.x, s1 * p02.y, s1 * p02.z, s1 * p02.w);
                const float4 u2 = make_float4(s2 * p01.x, s2 * p01.y, s2 * p01.z, s2 * p01.w);
                const bool fl0 = c[0] != cur0;
                red_add4_if(rowC(cur0), acc0, fl0 && cur0 >= 0);
                acc0 = fl0 ? u0 : make_float4(acc0.x + u0.x, acc0.y + u0.y, acc0.z + u0.z, acc0.w + u0.w);
                cur0 = c[0];
                if (POS1) {
                    const bool fl1 = c[1] != cur1;
                    red_add4_if(rowC(cur1), acc1, fl1 && has1);
                    const float4 base = fl1 ? make_float4(0, 0, 0, 0) : acc1;
                    acc1 = f1 ? make_float4(base.x + u1.x, base.y + u1.y, base.z + u1.z, base.w + u1.w) : base;
                    has1 = fl1 ? f1 : (has1 || f1);
                    cur1 = c[1];
                } else {
                    red_add4_if(rowC(c[1]), u1, f1);
                }
                red_add4_if(rowC(c[2]), u2, f2);
            }
        }
        // flush this group's pending sums at every chunk end
        red_add4_if(rowC(cur0), acc0, cur0 >= 0);
        cur0 = -1;
        if (POS1) {
            red_add4_if(rowC(cur1), acc1, has1);
            has1 = false;
            cur1 = -1;
        }
        __syncwarp();
    }
}

using EncodeFn = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                              const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
    static EncodeFn fn = [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return static_cast<EncodeFn>(nullptr);
        return reinterpret_cast<EncodeFn>(p);
    }();
    return fn;
}

}  // namespace

// returns cudaErrorNotSupported when the shape is not the experiment's
cudaError_t launch_mttkrp_tma(Plan &p, const float *B, int R, float *C, int depth, bool pos1, int copies,
                              int64_t plane, cudaStream_t s) {
    if (p.order != 3 || R % 32 != 0 || reinterpret_cast<uintptr_t>(B) % 16 || reinterpret_cast<uintptr_t>(C) % 16)
        return cudaErrorNotSupported;
    EncodeFn enc = encode_fn();
    if (!enc) return cudaErrorNotSupported;
    TmaParams P{};
    const cuuint64_t gdim[2] = {static_cast<cuuint64_t>(R), static_cast<cuuint64_t>(p.dim)};
    const cuuint64_t gstride[1] = {static_cast<cuuint64_t>(R) * 4};
    const cuuint32_t box[2] = {32, 1};
    const cuuint32_t estr[2] = {1, 1};
    if (enc(&P.tmB, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(B), gdim, gstride, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return cudaErrorInvalidValue;
    const int K = 33, S = 2, wpb = 8;
    const int CH = 4 * K;
    const size_t stream_bytes = static_cast<size_t>(wpb) * S * 4 * CH * 4;
    const size_t smem = ((stream_bytes + 127) & ~size_t(127)) + static_cast<size_t>(wpb) * depth * 12 * 128 +
                        static_cast<size_t>(wpb) * (S + depth) * 8;
    void (*fn)(TmaParams);
    if (depth == 2) fn = pos1 ? mttkrp3_tma_kernel<true, 2> : mttkrp3_tma_kernel<false, 2>;
    else if (depth == 4) fn = pos1 ? mttkrp3_tma_kernel<true, 4> : mttkrp3_tma_kernel<false, 4>;
    else fn = pos1 ? mttkrp3_tma_kernel<true, 8> : mttkrp3_tma_kernel<false, 8>;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 148, occ = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, wpb * 32, smem)) != cudaSuccess) return e;
    occ = std::max(occ, 1);
    const int64_t total_warps = static_cast<int64_t>(sms) * occ * wpb;
    int64_t span = (p.nnz + total_warps - 1) / total_warps;
    span = std::max<int64_t>(4, (span + 3) & ~3ll);
    const int64_t blocks = ((p.nnz + span - 1) / span + wpb - 1) / wpb;
    P.coords = p.coords;
    P.vals = p.vals;
    P.C = C;
    P.ld = p.ld;
    P.nnz = p.nnz;
    P.span = span;
    P.R = static_cast<uint32_t>(R);
    P.K = K;
    P.stages = S;
    P.copies = copies;
    P.plane = plane;
    fn<<<dim3(static_cast<unsigned>(blocks), static_cast<unsigned>(R / 32)), wpb * 32, smem, s>>>(P);
    p.last_grid_x = static_cast<int>(blocks);
    p.last_grid_y = R / 32;
    p.last_block = wpb * 32;
    p.last_smem = static_cast<int>(smem);
    return cudaGetLastError();
}

}  // namespace systec
