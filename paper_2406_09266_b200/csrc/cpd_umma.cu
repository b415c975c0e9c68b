// cpd_umma.cu — the CP-ALS dense pass at R = 32 on the 5th-generation tensor
// cores (tcgen05.mma kind::tf32, accumulators in TMEM; cpd.cu has the
// iteration it belongs to and the legacy mma.sync form, pass_tc32_kernel).
// Opt-in (SYSTEC_CPD_UMMA=1) and parity-tested against fp64 and the mma.sync
// form (tests/test_gpu_parity.py::test_cpd_pass_forms_vs_fp64): measured
// SLOWER on c3 (127 vs 101 us, profiles/r02/cpd_pass_umma_vs_mmasync.txt).
// The pass moves 48 KB of HBM per 128-row tile, but the 3xTF32 split needs
// the lo tiles and a K-major copy of M in shared memory besides the TMA tiles
// (~64 KB of converter writes), and the MMAs read ~144 KB of operands from
// shared memory per tile — about 270 KB of shared-memory traffic per tile,
// at 128 B/clk more than the tile's HBM time — with only two 96 KB stages
// in the 227 KB.  The mma.sync form reads each staged tile from shared memory
// once into registers.
//
// Per 128-row tile of M (the MTTKRP output) and F (the stored factor), with
// fp32 = hi + lo split into two TF32 operands (hi = tf32_rna(x), lo = x - hi;
// 3xTF32: a b ~ a_hi b_hi + a_hi b_lo + a_lo b_hi):
//   * Gram + fit dots in ONE M = 128, N = 64, K = 128 product:
//       A = [Mh | Ml | Fh | Fl]^T (128 x K, MN-major),  B = [Mh | Ml] (N = 64, MN-major)
//       D rows  0-31: [Mh^T Mh | Mh^T Ml]   rows 32-63: [Ml^T Mh | .]
//       D rows 64-95: [Fh^T Mh | Fh^T Ml]   rows 96-127: [Fl^T Mh | .]
//     so M^T M ~ D[0:32, 0:32] + D[0:32, 32:64] + D[32:64, 0:32] and the dots
//     sum_i F o M ~ diag of the three matching blocks of rows 64-127;
//   * F_new = M W (M = 128 rows, N = 32, K = 96): A = [Mh | Mh | Ml] (K-major),
//     B = [Wh ; Wl ; Wh] (K-major, W^T rows), stored over F's rows.
// Layouts: tiles arrive by TMA in the 128-byte swizzle with 32-byte atoms
// (SWIZZLE_128B_ATOM_32B: the only shared-memory layout the tensor cores take
// for MN-major TF32 operands — with the plain 128-byte swizzle they read
// zeros, measured), which is the Gram's MN-major view (rows = K, columns =
// MN); M W needs M K-major (rows = M, columns = K, 128-byte swizzle with
// 16-byte atoms), so the converters also write M's hi/lo in that layout.
//
// Warp roles (one CTA per SM, tiles b, b + grid, ...):
//   warp 0      TMA producer: M and F tiles into a 2-stage ring (96 KB each:
//               Mh | Ml | Fh | Fl MN-major, Mh | Ml K-major), zero rows past
//               dim (tensor-map OOB fill);
//   warp 1      TMEM allocation and the MMA issuer (one thread): 16 Gram MMAs
//               and 12 apply MMAs per tile into double-buffered TMEM
//               accumulators, tcgen05.commit to the stage's "empty" and the
//               buffer's "done" barriers;
//   warps 4-7   converters: hi/lo split (hi in place, lo beside it, and M's
//               K-major copies; generic-proxy writes, then fence.proxy.async
//               before arriving on the stage's barrier);
//   warps 8-11  epilogue (TMEM lane quadrant = warp % 4): tcgen05.ld of the
//               tile's F_new rows (stored to global) and Gram rows (added to
//               fp64 registers: fp32 inside a tile's 128 rows, fp64 across).
#include <cuda.h>

#include <algorithm>
#include <cstdlib>

#include "internal.cuh"
#include "ptx.cuh"

namespace systec {
namespace {

constexpr int kR = 32;
constexpr int kRows = 128;                      // tile rows
constexpr int kTileBytes = kRows * kR * 4;      // 16 KB
constexpr int kStageBytes = 6 * kTileBytes;     // Mh | Ml | Fh | Fl (MN-major) | Mh | Ml (K-major)
constexpr int kStages = 2;
constexpr int kWBytes = kR * kR * 4;            // 4 KB: W^T hi or lo
constexpr int kThreads = 384;
constexpr int kTmemCols = 256;                  // 2 x (64 Gram + 32 apply) columns, power of 2
constexpr size_t kSmemBytes = 1024 + static_cast<size_t>(kStages) * kStageBytes + 2 * kWBytes + 256;


// ---- tcgen05 / TMA wrappers ---------------------------------------------------
__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *tm, int c0, int c1, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
            "r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
// shared-memory matrix descriptor, 128-byte swizzle (sm_100: version 1, layout type 2)
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint64_t layout = 2) {
    return static_cast<uint64_t>((saddr >> 4) & 0x3FFFu) | (static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16) |
           (static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46) | (layout << 61);
}
// instruction descriptor, kind::tf32: D f32, A/B tf32, majors (0 = K, 1 = MN), N >> 3, M >> 4
constexpr uint32_t idesc_tf32(int M, int N, int amaj, int bmaj) {
    return (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(amaj) << 15) |
           (static_cast<uint32_t>(bmaj) << 16) | (static_cast<uint32_t>(N >> 3) << 17) |
           (static_cast<uint32_t>(M >> 4) << 24);
}
__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, int accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t *bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
// 32 lanes x 32 consecutive fp32 columns: thread = lane, v[j] = column j
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
}
__device__ __forceinline__ float tf32_rna(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

__global__ void __launch_bounds__(kThreads, 1) pass_umma32_kernel(const __grid_constant__ CUtensorMap tmM,
                                                                  const __grid_constant__ CUtensorMap tmF,
                                                                  float *F, const float *__restrict__ W,
                                                                  int64_t dim, double *__restrict__ part, int store,
                                                                  const int *skip) {
    extern __shared__ unsigned char umma_smem_raw[];
    // 1024-byte aligned base (the 128-byte swizzle repeats every 1024 bytes)
    unsigned char *smem = reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(umma_smem_raw) + 1023) &
                                                            ~static_cast<uintptr_t>(1023));
    unsigned char *stage0 = smem;
    unsigned char *wh = smem + static_cast<size_t>(kStages) * kStageBytes;
    unsigned char *wl = wh + kWBytes;
    uint64_t *bars = reinterpret_cast<uint64_t *>(wl + kWBytes);
    uint64_t *full = bars, *conv = bars + kStages, *empty = bars + 2 * kStages;
    uint64_t *done = bars + 3 * kStages, *tfree = done + 2;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tfree + 2);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const bool write = store && !(skip && *skip);
    const int64_t tiles = (dim + kRows - 1) / kRows;
    const int64_t nk = tiles > blockIdx.x ? (tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;

    // W^T hi / lo as K-major B operands: row n (128 B) holds W[k][n], k = 0..31,
    // its 16-byte chunks XOR-swizzled by (n % 8)
    for (int q = tid; q < kR * kR; q += kThreads) {
        const int n = q / kR, k = q % kR;
        const float w = W[k * kR + n];
        const float h = tf32_rna(w);
        const uint32_t off = static_cast<uint32_t>(n * 128 + ((k * 4) ^ ((n & 7) << 4)));
        *reinterpret_cast<float *>(wh + off) = h;
        *reinterpret_cast<float *>(wl + off) = w - h;
    }
    if (tid == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&conv[s], 128);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&done[b], 1);
            mbar_init(&tfree[b], 128);
        }
        fence_mbar_init();
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(kTmemCols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    fence_proxy_async_smem();  // the W tiles (generic writes) are read by the tensor cores
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            for (int64_t k = 0; k < nk; ++k) {
                const int s = static_cast<int>(k % kStages);
                if (k >= kStages) mbar_wait(&empty[s], static_cast<uint32_t>((k / kStages - 1) & 1));
                unsigned char *st = stage0 + static_cast<size_t>(s) * kStageBytes;
                const int row0 = static_cast<int>((blockIdx.x + k * gridDim.x) * kRows);
                mbar_arrive_expect_tx(&full[s], 2 * kTileBytes);
                tma_load_2d(st, &tmM, 0, row0, &full[s]);
                tma_load_2d(st + 2 * kTileBytes, &tmF, 0, row0, &full[s]);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t kIdGram = idesc_tf32(128, 64, 1, 1);
            constexpr uint32_t kIdApply = idesc_tf32(128, 32, 0, 0);
            const uint32_t wh_a = smem_u32(wh), wl_a = smem_u32(wl);
            for (int64_t k = 0; k < nk; ++k) {
                const int s = static_cast<int>(k % kStages);
                const int b = static_cast<int>(k & 1);
                mbar_wait(&conv[s], static_cast<uint32_t>((k / kStages) & 1));
                if (k >= 2) mbar_wait(&tfree[b], static_cast<uint32_t>((k / 2 - 1) & 1));
                tc_fence_after();
                const uint32_t st = smem_u32(stage0 + static_cast<size_t>(s) * kStageBytes);
                const uint32_t tg = tmem + static_cast<uint32_t>(b * 96);  // Gram: 64 columns
                const uint32_t ta = tg + 64;                                // apply: 32 columns
                // Gram + dots: K = the tile's 128 rows, 8 per MMA (one 1024-byte row group)
#pragma unroll 1
                for (int kk = 0; kk < kRows / 8; ++kk) {
                    // MN-major, 128-byte swizzle with 32-byte atoms: atoms of 4 rows
                    // (SBO 512 B), the four 32-column blocks 16 KB apart (LBO)
                    const uint64_t d = sdesc(st + kk * 1024, kTileBytes, 512, 1);
                    umma_tf32(tg, d, d, kIdGram, kk > 0);
                }
                if (write) {
                    // F_new = Mh Wh + Mh Wl + Ml Wh, K = 32 per product, 8 per MMA (32 bytes)
#pragma unroll 1
                    for (int pr = 0; pr < 3; ++pr) {
                        const uint32_t am = st + 4 * kTileBytes + (pr == 2 ? kTileBytes : 0);
                        const uint32_t bw = pr == 1 ? wl_a : wh_a;
#pragma unroll
                        for (int ks = 0; ks < 4; ++ks)
                            umma_tf32(ta, sdesc(am + ks * 32, 16, 1024), sdesc(bw + ks * 32, 16, 1024), kIdApply,
                                      pr > 0 || ks > 0);
                    }
                }
                umma_commit(&empty[s]);
                umma_commit(&done[b]);
            }
        }
    } else if (warp >= 4 && warp < 8) {
        const int ct = tid - 128;
        for (int64_t k = 0; k < nk; ++k) {
            const int s = static_cast<int>(k % kStages);
            mbar_wait(&full[s], static_cast<uint32_t>((k / kStages) & 1));
            unsigned char *st = stage0 + static_cast<size_t>(s) * kStageBytes;
#pragma unroll
            for (int m = 0; m < 2; ++m) {  // M, F: hi in place, lo into the next tile
                float4 *hi = reinterpret_cast<float4 *>(st + m * 2 * kTileBytes);
                float4 *lo = reinterpret_cast<float4 *>(st + m * 2 * kTileBytes + kTileBytes);
                float4 x[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) x[u] = hi[u * 128 + ct];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int q = u * 128 + ct;  // 16-byte chunk of the tile
                    const float4 h = make_float4(tf32_rna(x[u].x), tf32_rna(x[u].y), tf32_rna(x[u].z), tf32_rna(x[u].w));
                    const float4 l = make_float4(x[u].x - h.x, x[u].y - h.y, x[u].z - h.z, x[u].w - h.w);
                    hi[q] = h;
                    lo[q] = l;
                    if (m == 0) {
                        // row r, physical 32-byte atom of the chunk -> logical 16-byte
                        // chunk lc (columns 4 lc .. 4 lc + 3) -> its K-major place
                        const int r = q >> 3;
                        const int lc = ((((q & 7) >> 1) ^ (r & 3)) << 1) | (q & 1);
                        const int kq = r * 8 + (lc ^ (r & 7));
                        reinterpret_cast<float4 *>(st + 4 * kTileBytes)[kq] = h;
                        reinterpret_cast<float4 *>(st + 5 * kTileBytes)[kq] = l;
                    }
                }
            }
            fence_proxy_async_smem();
            mbar_arrive(&conv[s]);
        }
    } else if (warp >= 8) {
        const int quad = warp & 3;  // TMEM lanes [32 quad, 32 quad + 32)
        const int row = quad * 32 + lane;
        double gacc[32];
#pragma unroll
        for (int c = 0; c < 32; ++c) gacc[c] = 0.0;
        double dacc = 0.0;
        for (int64_t k = 0; k < nk; ++k) {
            const int b = static_cast<int>(k & 1);
            mbar_wait(&done[b], static_cast<uint32_t>((k / 2) & 1));
            tc_fence_after();
            const uint32_t tg = tmem + static_cast<uint32_t>(b * 96) + (static_cast<uint32_t>(quad * 32) << 16);
            if (write) {
                float v[32];
                tmem_ld32(tg + 64, v);
                const int64_t g = (blockIdx.x + k * gridDim.x) * kRows + row;
                if (g < dim) {
                    float4 *o = reinterpret_cast<float4 *>(F + g * kR);
#pragma unroll
                    for (int j = 0; j < 8; ++j) o[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
                }
            }
            float u[32], w[32];
            tmem_ld32(tg, u);
            tmem_ld32(tg + 32, w);
            tc_fence_before();
            mbar_arrive(&tfree[b]);
            if (quad == 0) {  // Mh^T rows: both column blocks are Gram terms
#pragma unroll
                for (int c = 0; c < 32; ++c) gacc[c] += static_cast<double>(u[c]) + static_cast<double>(w[c]);
            } else if (quad == 1) {  // Ml^T rows: the Ml^T Mh block
#pragma unroll
                for (int c = 0; c < 32; ++c) gacc[c] += static_cast<double>(u[c]);
            } else {  // F^T rows: the diagonal (column = lane) of the matching blocks
                float d = 0.f;
#pragma unroll
                for (int c = 0; c < 32; ++c)
                    if (c == lane) d = quad == 2 ? u[c] + w[c] : u[c];
                dacc += static_cast<double>(d);
            }
        }
        // per-block partial {M^T M, dots}: rows of quad 0 plus rows of quad 1,
        // dots of quad 2 plus quad 3, in a fixed order (named barrier 1: the
        // epilogue warps; the ring is idle — every tile's MMAs have completed)
        double *red = reinterpret_cast<double *>(stage0);  // [R][R], then [R] dots
        double *dred = red + kR * kR;
        if (quad == 0) {
#pragma unroll
            for (int c = 0; c < 32; ++c) red[lane * kR + c] = gacc[c];
        } else if (quad == 2) {
            dred[lane] = dacc;
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (quad == 1) {
#pragma unroll
            for (int c = 0; c < 32; ++c) red[lane * kR + c] += gacc[c];
        } else if (quad == 3) {
            dred[lane] += dacc;
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
        double *out = part + static_cast<int64_t>(blockIdx.x) * (kR * kR + kR);
        const int et = tid - 256;
        for (int q = et; q < kR * kR + kR; q += 128) out[q] = q < kR * kR ? red[q] : dred[q - kR * kR];
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols) : "memory");
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

// X [dim][32] fp32 as a 2-D tensor {32, dim}, 128 x 32 boxes, 128-byte
// swizzle with 32-byte atoms, rows past dim read as zeros
bool encode_rows32(CUtensorMap *tm, const float *X, int64_t dim) {
    EncodeFn enc = encode_fn();
    if (!enc) return false;
    const cuuint64_t gdim[2] = {static_cast<cuuint64_t>(kR), static_cast<cuuint64_t>(dim)};
    const cuuint64_t gstride[1] = {static_cast<cuuint64_t>(kR) * 4};
    const cuuint32_t box[2] = {static_cast<cuuint32_t>(kR), static_cast<cuuint32_t>(kRows)};
    const cuuint32_t estr[2] = {1, 1};
    return enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(X), gdim, gstride, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

int cpd_umma_blocks(int64_t dim) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t tiles = (dim + kRows - 1) / kRows;
    return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(sms, tiles)));
}

cudaError_t launch_pass_umma32(const float *M, float *F, const float *W, int64_t dim, double *part, int store,
                               const int *skip, cudaStream_t s) {
    if (dim < 1 || dim > 0x7FFFFFFF - kRows || (reinterpret_cast<uintptr_t>(M) & 15) ||
        (reinterpret_cast<uintptr_t>(F) & 15))
        return cudaErrorNotSupported;
    CUtensorMap tmM, tmF;
    if (!encode_rows32(&tmM, M, dim) || !encode_rows32(&tmF, F, dim)) return cudaErrorNotSupported;
    cudaError_t e = cudaFuncSetAttribute(pass_umma32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(kSmemBytes));
    if (e != cudaSuccess) return e;
    pass_umma32_kernel<<<cpd_umma_blocks(dim), kThreads, kSmemBytes, s>>>(tmM, tmF, F, W, dim, part, store, skip);
    return cudaGetLastError();
}

}  // namespace systec
