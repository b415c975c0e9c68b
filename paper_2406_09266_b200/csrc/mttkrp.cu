// mttkrp.cu — host-side launch of the symmetric MTTKRP kernel (see
// mttkrp_kernel.cuh for what the kernel computes and how it maps to sm_100a).
// Chooses the lane geometry for R, sizes the persistent grid from the
// occupancy calculator (a multiple of the 148 SMs), zeroes C and launches.
#include <algorithm>

#include "mttkrp_kernel.cuh"

namespace systec {

namespace {

KernelFn pick_naive(int order, int vw, int lpe, bool pf) {
    switch (order) {
        case 2: return pick_naive_kernel<2>(vw, lpe, pf);
        case 3: return pick_naive_kernel<3>(vw, lpe, pf);
        case 4: return pick_naive_kernel<4>(vw, lpe, pf);
        case 5: return pick_naive_kernel<5>(vw, lpe, pf);
        default: return nullptr;
    }
}

KernelFn pick(int order, int vw, int lpe, int vpl, bool pos1, bool pf) {
    switch (order) {
        case 2: return pick_kernel<2>(vw, lpe, vpl, pos1, pf);
        case 3: return pick_kernel<3>(vw, lpe, vpl, pos1, pf);
        case 4: return pick_kernel<4>(vw, lpe, vpl, pos1, pf);
        case 5: return pick_kernel<5>(vw, lpe, vpl, pos1, pf);
        default: return nullptr;
    }
}

KernelFn pick_full_naive(int order, int lpe) {
    switch (order) {
        case 3: return pick_full_naive_kernel<3>(lpe);
        case 4: return pick_full_naive_kernel<4>(lpe);
        case 5: return pick_full_naive_kernel<5>(lpe);
        default: return nullptr;
    }
}

KernelFn pick_full(int order, int lpe, bool pos1, bool occ) {
    switch (order) {
        case 3: return pick_full_kernel<3>(lpe, pos1, occ);
        case 4: return pick_full_kernel<4>(lpe, pos1, occ);
        case 5: return pick_full_kernel<5>(lpe, pos1, occ);
        default: return nullptr;
    }
}

int pow2ceil(int x) {
    int p = 1;
    while (p < x) p <<= 1;
    return p;
}

// Entries per lane group per chunk: odd for E >= 4 (the E groups then read
// distinct shared-memory banks) with E*K a multiple of 4 (16-byte copies);
// CH = E*K stays ~128-160 entries whatever the lane geometry.
int default_K(int E) {
    switch (E) {
        case 1: return 128;
        case 2: return 64;
        case 4: return 33;
        case 8: return 17;
        case 16: return 9;
        default: return 5;
    }
}

}  // namespace

KernelFn ablation3(int abl);
KernelFn ablation5(int abl);
KernelFn pick_ablation_kernel(int order, int abl) {
    return order == 3 ? ablation3(abl) : order == 5 ? ablation5(abl) : nullptr;
}

// Sum `copies` replicas Cp[copies][plane] into C[plane].  Groups of G lanes
// share one float4 of the plane, lane k adding replicas k, k+G, ... (more
// loads in flight than one thread per float4), then a shuffle reduction in
// fixed order; accumulate != 0 adds the result to C's contents.
template <int G>
__global__ void reduce_copies_kernel(const float *__restrict__ Cp, float *__restrict__ C, int64_t plane, int copies,
                                     int vec, int accumulate) {
    const int64_t n4 = vec ? plane / 4 : 0;
    const float4 *P4 = reinterpret_cast<const float4 *>(Cp);
    float4 *C4 = reinterpret_cast<float4 *>(C);
    const int k = threadIdx.x % G;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * (blockDim.x / G);
    // block-uniform loop bound: every lane reaches the shuffles
    for (int64_t base = blockIdx.x * static_cast<int64_t>(blockDim.x / G); base < n4; base += stride) {
        const int64_t i = base + threadIdx.x / G;
        const bool valid = i < n4;
        float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int c = k; valid && c < copies; c += G) {
            const float4 b = P4[c * n4 + i];
            a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
        }
#pragma unroll
        for (int d = G / 2; d > 0; d >>= 1) {
            a.x += __shfl_xor_sync(0xffffffffu, a.x, d, G);
            a.y += __shfl_xor_sync(0xffffffffu, a.y, d, G);
            a.z += __shfl_xor_sync(0xffffffffu, a.z, d, G);
            a.w += __shfl_xor_sync(0xffffffffu, a.w, d, G);
        }
        if (k == 0 && valid) {
            if (accumulate) {
                const float4 c = C4[i];
                a.x += c.x; a.y += c.y; a.z += c.z; a.w += c.w;
            }
            C4[i] = a;
        }
    }
    for (int64_t i = 4 * n4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < plane;
         i += (int64_t)gridDim.x * blockDim.x) {
        float a = accumulate ? C[i] : 0.f;
        for (int c = 0; c < copies; ++c) a += Cp[c * plane + i];
        C[i] = a;
    }
}

// L2-slice spreading: an output smaller than ~4 MB maps onto a few L2 slices
// whose atomic units then serialise the reductions (ncu on c5: atomic-input
// activity max 57 % vs avg 20 %); spread it over replicas.
static int replica_count(const Plan &p, int R, const systec_exec_opts &o) {
    const int64_t plane = p.dim * static_cast<int64_t>(R);
    int copies = o.copies;
    if (copies <= 0) {
        const int64_t bytes = plane * 4;
        copies = bytes >= (4 << 20) ? 1 : static_cast<int>(std::min<int64_t>(32, (4 << 20) / std::max<int64_t>(bytes, 1)));
        if (p.nnz < 100000) copies = 1;  // latency-bound sizes: not worth the extra pass
    }
    return copies;
}

// work counters of the dynamic distribution: one per rank tile (blockIdx.y);
// a tile is at least 32 columns wide, so ceil(R/32) bounds their number
static int64_t counter_slots(int R) { return ((R + 31) / 32 + 3) & ~3; }

// Scratch of one launch (floats): the C replicas when copies > 1, then the
// work counters of the dynamic distribution.
int64_t mttkrp_scratch_floats(const Plan &p, int R, const systec_exec_opts &o) {
    const int copies = replica_count(p, R, o);
    const int64_t rep = copies > 1 ? static_cast<int64_t>(copies) * p.dim * R : 0;
    return rep + (o.static_ranges > 0 ? 0 : counter_slots(R));
}

// C = 0 (16-byte stores when aligned) and the work counters = 0, one launch
__global__ void zero_output_kernel(float *__restrict__ C, int64_t plane, int vec, unsigned int *ctr, int nctr) {
    if (ctr && blockIdx.x == 0)
        for (int q = threadIdx.x; q < nctr; q += blockDim.x) ctr[q] = 0u;
    const int64_t n4 = vec ? plane / 4 : 0;
    float4 *C4 = reinterpret_cast<float4 *>(C);
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n4; i += stride)
        C4[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int64_t i = 4 * n4 + blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < plane; i += stride)
        C[i] = 0.f;
}

cudaError_t launch_mttkrp(const Plan &p, const float *B, int R, float *C, const systec_exec_opts &o, cudaStream_t s,
                          float *scratch_in) {
    cudaError_t e;
    // order 2: the atomic-free windowed kernel writes every row of C once (no zeroing pass)
    if (p.order == 2 && !p.general && o.window >= 0 && p.win_capp > 0 && o.ablation <= 0 && !o.force_scalar) {
        e = launch_sym2_window(p, B, R, C, o.no_zero != 0, s);
        if (e != cudaErrorNotSupported) return e;
        cudaGetLastError();
    }
    const int64_t plane = p.dim * static_cast<int64_t>(R);
    const int copies = replica_count(p, R, o);
    if (copies > 64) return cudaErrorInvalidValue;
    // work distribution: dynamic units from a counter (default) or one static
    // range per warp (opts.static_ranges = 1; measured: c3 2.43 -> 2.04 ms,
    // c4 -2 %, c5 -2 %, c2 -0.3 % with the dynamic one, profiles/r01_sweep_dynamic.jsonl)
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    // (a problem with fewer ~128-entry units than 8 warps per SM never runs dynamic: no counter)
    // dynamic units pay where the per-chunk work is large and the costs per
    // entry vary (orders >= 3 with float4 lanes); orders 2 and scalar ranks keep
    // the static split (order 2, dim 1e6, 10M nnz: R = 1 0.115 vs 0.123 ms,
    // R = 32 0.558 vs 0.568 ms static vs dynamic)
    // (the ablation builds keep the static split they were measured with)
    // (the naive kernel over an expanded tensor gets the same distribution:
    // it is the baseline of the paper's experiment, given its best form)
    const bool dyn = o.static_ranges <= 0 && o.ablation <= 0 && p.order >= 3 && R >= 8 &&
                     p.nnz / 128 >= static_cast<int64_t>(sms) * 8;
    const int64_t rep_f = copies > 1 ? static_cast<int64_t>(copies) * plane : 0;
    const int64_t nctr = dyn ? counter_slots(R) : 0;
    const int64_t need_f = rep_f + nctr;
    float *Cdst = C;
    float *scratch = nullptr;
    const bool own_scratch = scratch_in == nullptr;  // else: caller-provided (allocation-free launch)
    if (need_f > 0) {
        if (own_scratch) {
            e = cudaMallocAsync(&scratch, static_cast<size_t>(need_f) * 4, s);  // stream-ordered pool
            if (e != cudaSuccess) return e;
        } else {
            scratch = scratch_in;
        }
    }
    unsigned int *ctr = dyn ? reinterpret_cast<unsigned int *>(scratch + rep_f) : nullptr;
    if (copies > 1) {
        e = cudaMemsetAsync(scratch, 0, static_cast<size_t>(need_f) * 4, s);  // replicas (+ counter)
        if (e != cudaSuccess) return e;
        Cdst = scratch;
    } else if (!o.no_zero && !ctr) {
        e = cudaMemsetAsync(C, 0, static_cast<size_t>(plane) * sizeof(float), s);
        if (e != cudaSuccess) return e;
    } else if (!o.no_zero) {
        const int vec = (reinterpret_cast<uintptr_t>(C) % 16 == 0) ? 1 : 0;
        const int64_t work = std::max<int64_t>(1, vec ? plane / 4 : plane);
        const int zb = static_cast<int>(std::min<int64_t>((work + 255) / 256, static_cast<int64_t>(sms) * 8));
        zero_output_kernel<<<zb, 256, 0, s>>>(C, plane, vec, ctr, static_cast<int>(nctr));
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    } else if (ctr) {
        e = cudaMemsetAsync(ctr, 0, static_cast<size_t>(nctr) * sizeof(unsigned int), s);
        if (e != cudaSuccess) return e;
    }
    if (p.nnz == 0) {
        if (scratch && own_scratch) cudaFreeAsync(scratch, s);
        if (copies > 1 && !o.no_zero) return cudaMemsetAsync(C, 0, static_cast<size_t>(plane) * sizeof(float), s);
        return cudaSuccess;
    }

    const bool aligned = (reinterpret_cast<uintptr_t>(B) % 16 == 0) && (reinterpret_cast<uintptr_t>(C) % 16 == 0);
    auto release = [&](cudaError_t err) {
        if (scratch && own_scratch) cudaFreeAsync(scratch, s);
        return err;
    };
    const int vw = (R % 4 == 0 && aligned && !o.force_scalar) ? 4 : 1;
    const int vecs = (R + vw - 1) / vw;              // vectors per B row
    const int tile_vecs = std::min(32, pow2ceil(vecs));
    int vpl = 1;
    if (vw == 4 && !p.general) {
        const int want = o.vpl > 0 ? o.vpl : 1;  // float4 per lane
        vpl = std::min(want, tile_vecs);
        if (vpl != 1 && vpl != 2 && vpl != 4) return cudaErrorInvalidValue;
    }
    // 32-byte lanes (opts.lane_bytes = 32): the fixed-rank shapes with 8
    // columns per lane and one 256-bit gather per row — half the lanes per
    // entry, twice the entries per warp instruction
    const bool al32 = (reinterpret_cast<uintptr_t>(B) % 32 == 0) && (reinterpret_cast<uintptr_t>(C) % 32 == 0);
    const bool v8 = o.lane_bytes == 32 && al32 && vw == 4 && !p.general && o.fixed_rank >= 0 && o.vpl <= 1 &&
                    o.prefetch <= 0 && o.ablation <= 0 && o.occupancy <= 0 && o.chunk_k <= 0 &&
                    ((p.order == 3 && R == 32) || (p.order >= 4 && p.order <= 5 && R == 16));
    const int lpe = v8 ? R / 8 : tile_vecs / vpl;
    const int E = 32 / lpe;
    const int tiles = (R + tile_vecs * vw - 1) / (tile_vecs * vw);
    int K = o.chunk_k > 0 ? o.chunk_k : default_K(E);
    const int stages = o.stages > 0 ? o.stages : 2;
    if ((E * K) % 4 != 0 || stages > 8) return release(cudaErrorInvalidValue);

    bool pos1 = false;
    if (p.general) pos1 = false;  // the general kernel updates position 0 only
    else if (o.pos1_accumulate > 0) pos1 = true;
    else if (o.pos1_accumulate == 0 && p.stats.pos1_runs > 0)
        pos1 = (static_cast<double>(p.nnz) / static_cast<double>(p.stats.pos1_runs)) >= 1.5;

    // software-prefetch the next entry's B rows: opt-in.  Measured (profiles/
    // r01_sweep_v3.jsonl): c2 -1 %, c3 +12 %, c4/c5 +1 % time with the
    // branch-free kernel — the extra registers cost more occupancy than the
    // in-flight gathers gain.
    const bool pf = o.prefetch > 0;
    KernelFn fn = p.general ? pick_naive(p.order, vw, lpe, pf) : pick(p.order, vw, lpe, vpl, pos1, pf);
    // occupancy variant: 5 resident blocks (48 registers) for the order-3 R=32
    // kernel when B is too large to stay L2-resident and the stream is
    // lexicographic, so gathers wait on DRAM and more warps in flight pay
    // (c3 lexicographic: 2.65 -> 2.40 ms; c2 with its 12.8 MB B is
    // L2-resident and loses 2 %).  A banded plan (c3's default) keeps its
    // gathers in an L2 window and the 64-register fixed-rank kernel is faster
    // there (c3: 1.67-1.72 vs 1.73-1.76 ms, profiles/r02_c3_occupancy.jsonl).
    // opts.occupancy: 1 on, -1 off, 0 auto.
    const bool occ_shape = vw == 4 && vpl == 1 && !pf && !p.general &&
                           ((p.order == 3 && lpe == 8) || (p.order >= 4 && lpe == 4));
    const bool occ5 = occ_shape && (o.occupancy > 0 || (o.occupancy == 0 && p.order == 3 && p.band_shift < 0 &&
                                                         plane * 4 > (64ll << 20)));
    if (occ5) fn = p.order == 3 ? occupancy3(pos1) : p.order == 4 ? occupancy4(pos1) : occupancy5(pos1);
    // fixed-rank build when R is exactly one float4 tile of 16 or 32 columns
    // (opts.fixed_rank: 0 auto = on, -1 off)
    bool full = false;
    // (the naive kernel only on request, fixed_rank = 1: its general-rank build
    // measured as fast or faster — c4's expanded tensor 6.33 vs 8.70 ms,
    // profiles/r02/speedup_sym_vs_naive.jsonl)
    if (!v8 && (p.general ? o.fixed_rank > 0 : o.fixed_rank >= 0) && vw == 4 && vpl == 1 && !pf && tiles == 1 &&
        R == lpe * 4 &&
        o.ablation <= 0 && K == default_K(E)) {
        if (KernelFn ff = p.general ? pick_full_naive(p.order, lpe) : pick_full(p.order, lpe, pos1, occ5)) {
            fn = ff;
            full = true;
        }
    }
    if (v8) {
        fn = p.order == 3 ? pick_full_v8_kernel<3>(pos1) : p.order == 4 ? pick_full_v8_kernel<4>(pos1)
                                                                         : pick_full_v8_kernel<5>(pos1);
        full = true;
    }
    const int abl = o.ablation;
    if (abl > 0) {  // ablation study: only the c2 / c5 kernel shapes exist
        const bool shape3 = p.order == 3 && vw == 4 && lpe == 8 && vpl == 1 && !pos1 && !pf && !p.general;
        const bool shape5 = p.order == 5 && vw == 4 && lpe == 4 && vpl == 1 && pos1 && !pf && !p.general;
        fn = (shape3 || shape5) ? pick_ablation_kernel(p.order, abl) : nullptr;
    }
    if (!fn) return release(cudaErrorInvalidValue);
    int wpb = o.warps_per_block > 0 ? o.warps_per_block : 8;
    auto smem_for = [&](int w) {
        return static_cast<size_t>(w) * stages * (p.order + 1) * (E * K) * 4 + static_cast<size_t>(w) * stages * 24;
    };
    const size_t smem_cap = 200 * 1024;
    while (wpb > 1 && smem_for(wpb) > smem_cap) wpb >>= 1;  // keep the staging ring within shared memory
    if (smem_for(wpb) > smem_cap) return release(cudaErrorInvalidValue);
    const int threads = wpb * 32;
    const size_t smem = smem_for(wpb);
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return release(e);
    int occ = 1;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, threads, smem);
    if (e != cudaSuccess) return release(e);
    if (occ < 1) occ = 1;
    // L2-resident tables (B and C together <= 32 MB, unbanded): three blocks
    // per SM instead of four — fewer gathers and reductions in flight contend
    // less for the SM->L2 port when no row misses to DRAM (c2: 0.4753 vs
    // 0.4816 ms, reproducible; c3's DRAM misses want the fourth block: 1.84 vs
    // 1.65 ms with three).  opts.blocks_per_sm overrides.
    if (o.blocks_per_sm <= 0 && !p.general && p.order >= 3 && p.band_shift < 0 && 2 * plane * 4 <= (32ll << 20) &&
        occ > 3 && p.nnz >= 1000000)
        occ = 3;
    if (o.blocks_per_sm > 0) occ = std::min(occ, static_cast<int>(o.blocks_per_sm));
    const int64_t total_warps = static_cast<int64_t>(sms) * occ * wpb;
    int64_t span = (p.nnz + total_warps - 1) / total_warps;
    span = std::max<int64_t>(4, (span + 3) & ~3ll);
    const int64_t warps_used = (p.nnz + span - 1) / span;
    int64_t blocks = (warps_used + wpb - 1) / wpb;

    KParams kp;
    kp.coords = p.coords;
    kp.vals = p.vals;
    kp.B = B;
    kp.C = Cdst;
    kp.copies = copies;
    kp.plane = plane;
    kp.dim = p.dim;
    kp.ld = p.ld;
    kp.nnz = p.nnz;
    kp.span = span;
    kp.R = static_cast<uint32_t>(R);
    kp.K = K;
    kp.stages = stages;
    kp.hints = o.l2_hints >= 0 ? 1 : 0;
    kp.ctr = ctr;
    // unit size: one chunk balances best (c2 0.476 vs 0.486 ms with 4), but a
    // leading run spanning thousands of chunks (c3's hub row: 10M entries) is
    // then flushed by a different warp at every chunk — tens of thousands of
    // reductions into one row, serialised at its L2 slice (c3 2.69 vs 2.03 ms
    // with 4-chunk units).  SYSTEC_UNIT_CHUNKS overrides (measurements).
    static const int kUnitEnv = [] {
        const char *v = std::getenv("SYSTEC_UNIT_CHUNKS");
        const int u = v ? std::atoi(v) : 0;
        return u < 0 ? 0 : (u > 64 ? 64 : u);
    }();
    const bool big_b = p.dim * static_cast<int64_t>(R) * 4 > (64ll << 20);  // B (and C) not L2-resident
    // a banded stream (systec_plan_opts) takes 2-chunk units: c3 1.825 vs 1.85 ms
    // (4) / 1.92 (1), uniform dim-1e6 1.477 vs 1.485 / 1.772, dim-2^19 1.002 vs
    // 1.029 / 1.045 (profiles/r01_band_sweep5.jsonl)
    const int unit_chunks = kUnitEnv > 0 ? kUnitEnv
                            : p.band_shift >= 0 ? 2
                            : ((p.stats.max_lead_run > 4096ll * E * K || big_b) ? 4 : 1);
    kp.unit = E * K * unit_chunks;
    // problems with fewer units than resident warps (c1: 16 units) keep the
    // finer static split: more warps in flight beat balance there (c1 kernel
    // 6.2 vs 9.3 us)
    const int64_t units = (p.nnz + kp.unit - 1) / kp.unit;
    if (dyn && units >= total_warps) blocks = static_cast<int64_t>(sms) * occ;  // persistent
    else kp.ctr = nullptr;

    dim3 grid(static_cast<unsigned>(blocks), static_cast<unsigned>(tiles));
    fn<<<grid, threads, smem, s>>>(kp);
    if (copies > 1) {
        e = cudaGetLastError();
        if (e != cudaSuccess) return release(e);
        const int64_t work = std::max<int64_t>(1, plane / 4) * 8;  // 8 lanes per float4 of C
        const int rb = static_cast<int>(std::min<int64_t>((work + 255) / 256, static_cast<int64_t>(sms) * 8));
        const int vec = (reinterpret_cast<uintptr_t>(C) % 16 == 0) && (plane % 4 == 0);
        reduce_copies_kernel<8><<<rb, 256, 0, s>>>(scratch, C, plane, copies, vec, o.no_zero ? 1 : 0);
    }
    if (scratch && own_scratch) cudaFreeAsync(scratch, s);
    Plan::LaunchInfo li;
    li.grid_x = static_cast<int>(blocks);
    li.grid_y = tiles;
    li.block = threads;
    li.smem = static_cast<int>(smem);
    // kernel id, decimal fields: general | copies (2 digits) | pf + 2*dynamic | order | vw | lpe (2 digits) | vpl | pos1;
    // the occupancy variant sets vpl's digit to 5 (vpl itself is 1 there)
    li.kernel = (p.general ? 1000000000 : 0) + copies * 10000000 + ((pf ? 1 : 0) + (kp.ctr ? 2 : 0) + (full ? 4 : 0)) * 1000000 + p.order * 100000 + (v8 ? 8 : vw) * 10000 + lpe * 100 + (occ5 ? 5 : vpl) * 10 + (pos1 ? 1 : 0);
    p.record_launch(li);
    return cudaGetLastError();
}

}  // namespace systec
