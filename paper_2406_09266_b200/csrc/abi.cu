// abi.cu — the extern "C" boundary of libsystec (declared in include/systec.h).
// Argument checking, plan lifetime, stream-ordered memory and error mapping;
// every step of the computation itself runs in the kernels of prepare.cu and
// mttkrp.cu.  There is no host compute path.
#include <climits>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <new>
#include <vector>
#include <algorithm>
#include <atomic>
#include <mutex>

#include "internal.cuh"

static_assert(sizeof(systec_exec_opts) == 68, "systec_exec_opts layout is part of the ABI");
static_assert(sizeof(systec_stats) == 224, "systec_stats layout is part of the ABI");
static_assert(sizeof(systec_plan_opts) == 32, "systec_plan_opts layout is part of the ABI");

namespace systec {

static thread_local int g_last_cuda_error = 0;
static thread_local int64_t g_last_bad_entry = -1;
void set_last_cuda_error(cudaError_t e) { g_last_cuda_error = static_cast<int>(e); }

namespace {

int cuda_fail(cudaError_t e) {
    set_last_cuda_error(e);
    return e == cudaErrorMemoryAllocation ? SYSTEC_ERR_NOMEM : SYSTEC_ERR_CUDA;
}

int ceil_log2(int64_t dim) {
    int b = 0;
    while ((int64_t(1) << b) < dim) ++b;
    return b < 1 ? 1 : b;
}

bool overlap(const void *a, size_t na, const void *b, size_t nb) {
    if (!a || !b || na == 0 || nb == 0) return false;
    const uintptr_t x = reinterpret_cast<uintptr_t>(a), y = reinterpret_cast<uintptr_t>(b);
    return x < y + nb && y < x + na;
}

// Keep freed stream-ordered allocations in the current device's default pool
// (plans and replica scratch come from it), once per device, thread-safe.
void ensure_pool_keeps_memory() {
    static std::atomic<uint64_t> done_mask{0};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return;
    const uint64_t bit = 1ull << dev;
    if (done_mask.load(std::memory_order_acquire) & bit) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        if (cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr) == cudaSuccess)
            done_mask.fetch_or(bit, std::memory_order_acq_rel);
    }
}

int check_shape(int order, int64_t dim, int64_t nnz, int *bits_out) {
    if (dim < 1 || nnz < 0) return SYSTEC_ERR_ARG;
    if (order < 2 || order > 5) return SYSTEC_ERR_UNSUPPORTED;
    if (dim > INT32_MAX || nnz > INT32_MAX - 64) return SYSTEC_ERR_UNSUPPORTED;
    *bits_out = ceil_log2(dim);  // order * bits > 64: a wide plan (no packed 64-bit key; prepare.cu)
    return SYSTEC_OK;
}

void fill_stats(Plan *p, const DevStats &hst) {
    systec_stats &st = p->stats;
    st.G = static_cast<int64_t>(hst.G);
    st.expanded = static_cast<int64_t>(hst.expanded);
    for (int c = 0; c < 16; ++c) st.pattern_hist[c] = static_cast<int64_t>(hst.hist[c]);
    st.lead_runs = static_cast<int64_t>(hst.lead_runs);
    st.max_lead_run = static_cast<int64_t>(hst.max_lead_run);
    st.pos1_runs = static_cast<int64_t>(hst.pos1_runs);
}

// Band shift for a plan's stream order (systec_plan_opts.band_shift; -1 = lexicographic).
// Auto: order-3 symmetric plans with dim >= 2^19, i.e. B and C of at least
// 2 x 16 MB at R = 8 — c3 (dim 1e6, Zipf) runs 1.96 -> 1.82 ms with 16 bands,
// a uniform dim-1e6 order-3 tensor 1.62 -> 1.47 ms with 4; order 2 loses
// (its only reuse is the leading run, which bands cut) and is never banded
// automatically.  Bands: the largest power of two <= mean leading run / 5,
// at most 16 and at least 2^16 rows each (profiles/r01_band_sweep*.jsonl).
// One-shot calls (systec_mttkrp, systec_mttkrp_host) stay lexicographic: the
// re-sort is paid once per plan and pays back only over repeated executes.
int choose_band_shift(int request, int order, int64_t dim, int bits, int64_t nnz, int64_t lead_runs, bool general) {
    if (request < 0 || nnz < 2 || (general && request == 0)) return -1;
    int shift;
    if (request > 0) {
        shift = request;
    } else {
        if (order != 3 || dim < (int64_t(1) << 19) || lead_runs < 1) return -1;
        const double mean_run = static_cast<double>(nnz) / static_cast<double>(lead_runs);
        int bb = 0;
        while (bb < 4 && static_cast<double>(int64_t(2) << bb) <= mean_run / 5.0) ++bb;
        shift = std::max(bits - bb, 16);
    }
    if (shift >= 31) return -1;
    const int64_t bands = ((dim - 1) >> shift) + 1;
    if (bands < 2) return -1;
    return ceil_log2(bands) <= 16 ? shift : -1;  // band numbers are sorted as 16-bit keys
}

// Re-sorts a plan's prepared stream band-major: a stable radix sort of the
// entries' band numbers alone (the stream is already lexicographic, so one
// digit pass keeps that order within each band), then a permuting copy into
// new storage; refreshes the run statistics.
int apply_bands(Plan *p, int shift, bool pooled, cudaStream_t s) {
    const int64_t nnz = p->nnz;
    const size_t nk = static_cast<size_t>(nnz);
    const int band_bits = ceil_log2(((p->dim - 1) >> shift) + 1);
    const size_t bytes = static_cast<size_t>(p->order + 1) * p->ld * 4;
    void *storage = nullptr;
    DevStats *dst = nullptr;
    uint16_t *bk = nullptr, *bk2 = nullptr;
    uint32_t *perm = nullptr, *perm2 = nullptr;
    auto cleanup = [&]() {
        if (dst) cudaFreeAsync(dst, s);
        if (bk) cudaFreeAsync(bk, s);
        if (bk2) cudaFreeAsync(bk2, s);
        if (perm) cudaFreeAsync(perm, s);
        if (perm2) cudaFreeAsync(perm2, s);
    };
    auto fail = [&](cudaError_t err) {
        cleanup();
        if (storage) { if (pooled) cudaFreeAsync(storage, s); else cudaFree(storage); }
        return cuda_fail(err);
    };
    if (band_bits > 16) return SYSTEC_ERR_UNSUPPORTED;
    cudaError_t e = pooled ? cudaMallocAsync(&storage, bytes, s) : cudaMalloc(&storage, bytes);
    if (e != cudaSuccess) { storage = nullptr; return fail(e); }
    int32_t *coords = static_cast<int32_t *>(storage);
    float *vals = reinterpret_cast<float *>(coords + static_cast<size_t>(p->order) * p->ld);
    if ((e = cudaMallocAsync(&dst, sizeof(DevStats), s)) != cudaSuccess) return fail(e);
    if ((e = cudaMallocAsync(&bk, nk * 2, s)) != cudaSuccess) return fail(e);
    if ((e = cudaMallocAsync(&bk2, nk * 2, s)) != cudaSuccess) return fail(e);
    if ((e = cudaMallocAsync(&perm, nk * 4, s)) != cudaSuccess) return fail(e);
    if ((e = cudaMallocAsync(&perm2, nk * 4, s)) != cudaSuccess) return fail(e);
    if ((e = cudaMemsetAsync(dst, 0, sizeof(DevStats), s)) != cudaSuccess) return fail(e);
    if ((e = launch_band_keys(p->order, nnz, p->ld, p->coords, shift, bk, perm, s)) != cudaSuccess) return fail(e);
    if ((e = sort_band_keys(nnz, band_bits, bk, bk2, perm, perm2, s)) != cudaSuccess) return fail(e);
    if ((e = launch_permute(p->order, nnz, p->ld, perm2, p->coords, p->vals, coords, vals, s)) != cudaSuccess)
        return fail(e);
    if ((e = launch_stats(p->order, nnz, p->ld, coords, shift, dst, s)) != cudaSuccess) return fail(e);
    DevStats hst;
    if ((e = cudaMemcpyAsync(&hst, dst, sizeof(hst), cudaMemcpyDeviceToHost, s)) != cudaSuccess) return fail(e);
    cleanup();
    dst = nullptr; bk = nullptr; bk2 = nullptr; perm = nullptr; perm2 = nullptr;
    if (p->pooled) cudaFreeAsync(p->storage, s); else cudaFree(p->storage);
    p->storage = storage;
    p->coords = coords;
    p->vals = vals;
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return cuda_fail(e);  // the band statistics
    fill_stats(p, hst);
    p->band_shift = shift;
    p->stats.band_shift = shift;
    return SYSTEC_OK;
}

void free_window(Plan *p, bool pooled, cudaStream_t s) {
    if (!p->win_rowptr) return;
    if (pooled) cudaFreeAsync(p->win_rowptr, s); else cudaFree(p->win_rowptr);
    p->win_rowptr = p->win_colptr = nullptr;
    p->win_capp = 0;
}

// Builds the plan.  `pooled` plans keep their storage in the stream-ordered pool.
int plan_create_impl(Plan **out, int order, int64_t dim, int64_t nnz, const int32_t *idx, const float *vals,
                     cudaStream_t s, bool pooled, bool general = false, int band_request = 0,
                     bool window = false) {
    NvtxRange nvtx_range_("systec_plan_create");
    *out = nullptr;
    int bits = 0;
    int rc = check_shape(order, dim, nnz, &bits);
    if (rc) return rc;
    if (nnz > 0 && (!idx || !vals)) return SYSTEC_ERR_ARG;
    ensure_pool_keeps_memory();

    Plan *p = new (std::nothrow) Plan();
    if (!p) return SYSTEC_ERR_NOMEM;
    p->order = order;
    p->dim = dim;
    p->nnz = nnz;
    p->ld = ((nnz + 3) & ~int64_t(3)) + 4;
    p->key_bits = bits;
    p->pooled = pooled;
    p->general = general;
    p->stream = s;
    const size_t bytes = static_cast<size_t>(order + 1) * p->ld * 4;
    cudaError_t e = pooled ? cudaMallocAsync(&p->storage, bytes, s) : cudaMalloc(&p->storage, bytes);
    if (e != cudaSuccess) {
        delete p;
        return cuda_fail(e);
    }
    p->coords = static_cast<int32_t *>(p->storage);
    p->vals = reinterpret_cast<float *>(p->coords + static_cast<size_t>(order) * p->ld);

    DevStats *dst = nullptr;
    unsigned long long *keys = nullptr, *keys2 = nullptr;
    uint32_t *perm = nullptr, *perm2 = nullptr;
    DevStats hst;
    auto cleanup = [&]() {
        if (dst) cudaFreeAsync(dst, s);
        if (keys) cudaFreeAsync(keys, s);
        if (keys2) cudaFreeAsync(keys2, s);
        if (perm) cudaFreeAsync(perm, s);
        if (perm2) cudaFreeAsync(perm2, s);
    };
    auto fail = [&](cudaError_t err) {
        cleanup();
        free_window(p, pooled, s);
        if (pooled) cudaFreeAsync(p->storage, s); else cudaFree(p->storage);
        delete p;
        return cuda_fail(err);
    };
    const size_t nk = static_cast<size_t>(nnz > 0 ? nnz : 1);
    if ((e = cudaMallocAsync(&dst, sizeof(DevStats), s)) != cudaSuccess) return fail(e);
    std::memset(&hst, 0, sizeof(hst));
    hst.bad_entry = ULLONG_MAX;
    const DevStats hst0 = hst;
    if ((e = cudaMemcpyAsync(dst, &hst0, sizeof(hst0), cudaMemcpyHostToDevice, s)) != cudaSuccess) return fail(e);

    // order-2 symmetric plans: the windowed kernel's row / column pointers and
    // bandwidth, read back with the statistics (sym2_window.cu)
    unsigned long long win_host[2] = {0, 0};  // {bandwidth, largest column count}
    int32_t win_items = 0;
    auto build_window = [&]() -> cudaError_t {
        if (!(order == 2 && !general && window)) return cudaSuccess;
        cudaError_t we;
        if (!p->win_rowptr) {
            const size_t wb = static_cast<size_t>(dim + 1) * 8 + 16;
            void *w = nullptr;
            if ((we = pooled ? cudaMallocAsync(&w, wb, s) : cudaMalloc(&w, wb)) != cudaSuccess) return we;
            p->win_rowptr = static_cast<int32_t *>(w);
            p->win_colptr = p->win_rowptr + (dim + 1);
        }
        auto *wv = reinterpret_cast<unsigned long long *>(p->win_colptr + (dim + 1));
        if ((we = win_build(*p, p->win_rowptr, p->win_colptr, wv, wv + 1, s)) != cudaSuccess) return we;
        if ((we = cudaMemcpyAsync(win_host, wv, 16, cudaMemcpyDeviceToHost, s)) != cudaSuccess) return we;
        return cudaMemcpyAsync(&win_items, p->win_colptr + dim, 4, cudaMemcpyDeviceToHost, s);
    };

    // a1 + a2 in one pass, for input already in storage order (the common case):
    // validation, canonical tuples written straight into the SoA stream, the
    // sortedness flag and the statistics — one kernel, one synchronisation.
    if ((e = launch_prepare_sorted(order, dim, nnz, p->ld, idx, vals, p->coords, p->vals, dst, s, !general)) !=
        cudaSuccess)
        return fail(e);
    if ((e = cudaMemcpyAsync(&hst, dst, sizeof(hst), cudaMemcpyDeviceToHost, s)) != cudaSuccess) return fail(e);
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return fail(e);  // sync 1: verdict + statistics
    // (a pass that also saw a disorder stopped early: its first bad entry need not be
    // the first one — the sorting path below validates every entry and reports)
    if (hst.err && hst.unsorted == 0) {
        g_last_bad_entry = static_cast<int64_t>(hst.bad_entry);
        cleanup();
        free_window(p, pooled, s);
        if (pooled) cudaFreeAsync(p->storage, s); else cudaFree(p->storage);
        delete p;
        return SYSTEC_ERR_INDEX;
    }
    const bool sorted = hst.unsorted == 0 || nnz < 2;
    if (!sorted) {
        // a1/a2, sorting path: pack keys (wide plans: none), lexicographic radix
        // sort, SoA gather through the permutation, statistics of the sorted stream
        const bool wide = bits * order > 64;
        if ((e = cudaMallocAsync(&keys, nk * 8, s)) != cudaSuccess) return fail(e);
        if ((e = cudaMallocAsync(&perm, nk * 4, s)) != cudaSuccess) return fail(e);
        if ((e = cudaMallocAsync(&keys2, nk * 8, s)) != cudaSuccess) return fail(e);
        if ((e = cudaMallocAsync(&perm2, nk * 4, s)) != cudaSuccess) return fail(e);
        if ((e = cudaMemcpyAsync(dst, &hst0, sizeof(hst0), cudaMemcpyHostToDevice, s)) != cudaSuccess) return fail(e);
        e = wide ? launch_validate_wide(order, dim, nnz, idx, perm, dst, s, !general)
                 : launch_canonicalize(order, dim, nnz, bits, idx, keys, perm, dst, s, !general);
        if (e != cudaSuccess) return fail(e);
        const uint32_t *sperm = perm2;
        if (wide) {
            uint32_t *sorted_perm = nullptr;
            if ((e = sort_wide(order, dim, nnz, bits, idx, keys, keys2, perm, perm2, &sorted_perm, s, !general)) !=
                cudaSuccess)
                return fail(e);
            sperm = sorted_perm;
        } else if ((e = sort_keys(nnz, bits * order, keys, keys2, perm, perm2, s)) != cudaSuccess) {
            return fail(e);
        }
        e = wide ? launch_gather_wide(order, nnz, p->ld, p->ld, dim, idx, sperm, vals, p->coords, p->vals, s, !general)
                 : launch_gather(order, nnz, p->ld, bits, keys2, sperm, vals, p->coords, p->vals, s);
        if (e != cudaSuccess) return fail(e);
        // (no reset here: the one-pass kernel stops at the first tile after a disorder is
        // published, so this path's validation verdict is the complete one; the
        // canonicalise kernels write only the verdict fields, the counters are still zero)
        if ((e = launch_stats(order, nnz, p->ld, p->coords, -1, dst, s)) != cudaSuccess) return fail(e);
        if ((e = cudaMemcpyAsync(&hst, dst, sizeof(hst), cudaMemcpyDeviceToHost, s)) != cudaSuccess) return fail(e);
    }
    if ((e = build_window()) != cudaSuccess) return fail(e);  // order-2 window plans only (reads the sorted stream)
    cleanup();
    dst = nullptr; keys = nullptr; keys2 = nullptr; perm = nullptr; perm2 = nullptr;
    // sync 2: only on the sorting path (its statistics) and for window plans
    if ((!sorted || p->win_rowptr) && (e = cudaStreamSynchronize(s)) != cudaSuccess) {
        free_window(p, pooled, s);
        if (pooled) cudaFreeAsync(p->storage, s); else cudaFree(p->storage);
        delete p;
        return cuda_fail(e);
    }
    if (hst.err) {  // sorting path: a bad index in a tile the one-pass kernel never reached
        g_last_bad_entry = static_cast<int64_t>(hst.bad_entry);
        free_window(p, pooled, s);
        if (pooled) cudaFreeAsync(p->storage, s); else cudaFree(p->storage);
        delete p;
        return SYSTEC_ERR_INDEX;
    }
    if (p->win_rowptr) {
        p->win_bw = static_cast<int64_t>(win_host[0]);
        p->win_capp = win_partition(dim, win_items, p->win_bw, static_cast<int64_t>(win_host[1]), &p->win_nblk);
    }
    systec_stats &st = p->stats;
    st.nnz = nnz;
    st.dim = dim;
    st.order = order;
    st.key_bits = bits;
    fill_stats(p, hst);
    st.input_was_sorted = sorted ? 1 : 0;
    st.band_shift = -1;
    st.bad_entry = -1;
    // banded stream order (a second device sort of the prepared stream)
    const int shift = choose_band_shift(band_request, order, dim, bits, nnz, st.lead_runs, general);
    if (shift >= 0 && (rc = apply_bands(p, shift, pooled, s)) != SYSTEC_OK) {
        free_window(p, pooled, s);
        if (pooled) cudaFreeAsync(p->storage, s); else cudaFree(p->storage);
        delete p;
        return rc;
    }
    if (shift >= 0) p->win_capp = 0;  // the windowed kernel needs the row-sorted stream
    st.bandwidth = p->win_rowptr ? p->win_bw : 0;
    st.window_blocks = p->win_capp > 0 ? p->win_nblk : 0;
    *out = p;
    return SYSTEC_OK;
}

int execute_impl(Plan *p, const float *B, int R, float *C, const systec_exec_opts *opts, cudaStream_t s) {
    NvtxRange nvtx_range_("systec_plan_execute");
    if (!p || !B || !C || R < 1) return SYSTEC_ERR_ARG;
    const size_t bytes = static_cast<size_t>(p->dim) * R * sizeof(float);
    if (overlap(B, bytes, C, bytes)) return SYSTEC_ERR_ALIAS;
    if (overlap(C, bytes, p->storage, static_cast<size_t>(p->order + 1) * p->ld * 4)) return SYSTEC_ERR_ALIAS;
    systec_exec_opts o;
    std::memset(&o, 0, sizeof(o));
    if (opts) o = *opts;
    if (o.warps_per_block < 0 || o.warps_per_block > 8 || o.blocks_per_sm < 0) return SYSTEC_ERR_ARG;
    cudaError_t e = launch_mttkrp(*p, B, R, C, o, s);
    if (e == cudaErrorInvalidValue) return SYSTEC_ERR_ARG;
    if (e != cudaSuccess) return cuda_fail(e);
    return SYSTEC_OK;
}

void destroy_impl(Plan *p) {
    if (!p) return;
    free_window(p, p->pooled, p->stream);
    if (p->pooled) cudaFreeAsync(p->storage, p->stream);
    else cudaFree(p->storage);
    delete p;
}

}  // namespace
}  // namespace systec

using systec::Plan;

extern "C" {

int systec_plan_create(systec_plan *out, int order, int64_t dim, int64_t nnz, const int32_t *idx,
                       const float *vals, systec_stream_t stream) {
    if (!out) return SYSTEC_ERR_ARG;
    Plan *p = nullptr;
    int rc = systec::plan_create_impl(&p, order, dim, nnz, idx, vals, reinterpret_cast<cudaStream_t>(stream), false);
    *out = reinterpret_cast<systec_plan>(p);
    return rc;
}

int systec_plan_create_ex(systec_plan *out, int order, int64_t dim, int64_t nnz, const int32_t *idx,
                          const float *vals, const systec_plan_opts *opts, systec_stream_t stream) {
    if (!out) return SYSTEC_ERR_ARG;
    *out = nullptr;
    int band = 0;
    bool general = false, window = false;
    if (opts) {
        if (opts->band_shift < -1 || opts->general < 0 || opts->general > 1 || opts->window < 0 || opts->window > 1)
            return SYSTEC_ERR_ARG;
        for (int r : opts->reserved)
            if (r) return SYSTEC_ERR_ARG;
        band = opts->band_shift;
        general = opts->general == 1;
        window = opts->window == 1;
    }
    Plan *p = nullptr;
    int rc = systec::plan_create_impl(&p, order, dim, nnz, idx, vals, reinterpret_cast<cudaStream_t>(stream), false,
                                      general, band, window);
    *out = reinterpret_cast<systec_plan>(p);
    return rc;
}

int systec_plan_create_general(systec_plan *out, int order, int64_t dim, int64_t nnz, const int32_t *idx,
                               const float *vals, systec_stream_t stream) {
    if (!out) return SYSTEC_ERR_ARG;
    Plan *p = nullptr;
    int rc = systec::plan_create_impl(&p, order, dim, nnz, idx, vals, reinterpret_cast<cudaStream_t>(stream), false,
                                      true);
    *out = reinterpret_cast<systec_plan>(p);
    return rc;
}

int systec_expand_symmetric(int order, int64_t dim, int64_t nnz, const int32_t *idx, const float *vals,
                            int64_t capacity, int32_t *out_idx, float *out_vals, int64_t *count,
                            systec_stream_t stream) {
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    int bits = 0;
    int rc = systec::check_shape(order, dim, nnz, &bits);
    if (rc) return rc;
    if (!count || (nnz > 0 && (!idx || !vals))) return SYSTEC_ERR_ARG;
    *count = 0;
    if (nnz == 0) return SYSTEC_OK;
    systec::DevStats *dst = nullptr;
    unsigned long long *sizes = nullptr, *offsets = nullptr;
    systec::DevStats hst;
    std::memset(&hst, 0, sizeof(hst));
    hst.bad_entry = ULLONG_MAX;
    cudaError_t e = cudaSuccess;
    auto done = [&](int status) {
        if (dst) cudaFreeAsync(dst, s);
        if (sizes) cudaFreeAsync(sizes, s);
        if (offsets) cudaFreeAsync(offsets, s);
        return status;
    };
    if ((e = cudaMallocAsync(&dst, sizeof(hst), s)) != cudaSuccess) return done(systec::cuda_fail(e));
    if ((e = cudaMallocAsync(&sizes, nnz * 8, s)) != cudaSuccess) return done(systec::cuda_fail(e));
    if ((e = cudaMallocAsync(&offsets, nnz * 8, s)) != cudaSuccess) return done(systec::cuda_fail(e));
    if ((e = cudaMemcpyAsync(dst, &hst, sizeof(hst), cudaMemcpyHostToDevice, s)) != cudaSuccess)
        return done(systec::cuda_fail(e));
    if ((e = systec::expand_count(order, dim, nnz, idx, sizes, offsets, dst, s)) != cudaSuccess)
        return done(systec::cuda_fail(e));
    unsigned long long last[2] = {0, 0};
    if ((e = cudaMemcpyAsync(&hst, dst, sizeof(hst), cudaMemcpyDeviceToHost, s)) != cudaSuccess ||
        (e = cudaMemcpyAsync(&last[0], offsets + nnz - 1, 8, cudaMemcpyDeviceToHost, s)) != cudaSuccess ||
        (e = cudaMemcpyAsync(&last[1], sizes + nnz - 1, 8, cudaMemcpyDeviceToHost, s)) != cudaSuccess ||
        (e = cudaStreamSynchronize(s)) != cudaSuccess)
        return done(systec::cuda_fail(e));
    if (hst.err) {
        systec::g_last_bad_entry = static_cast<int64_t>(hst.bad_entry);
        return done(SYSTEC_ERR_INDEX);
    }
    *count = static_cast<int64_t>(last[0] + last[1]);
    if (!out_idx && !out_vals) return done(SYSTEC_OK);  // count-only query
    if (!out_idx || !out_vals || capacity < *count) return done(SYSTEC_ERR_ARG);
    if ((e = systec::expand_write(order, nnz, idx, vals, offsets, out_idx, out_vals, s)) != cudaSuccess)
        return done(systec::cuda_fail(e));
    return done(SYSTEC_OK);
}

int systec_plan_minplus(systec_plan plan, const float *d, float *y, systec_stream_t stream) {
    Plan *p = reinterpret_cast<Plan *>(plan);
    if (!p || !d || !y) return SYSTEC_ERR_ARG;
    if (p->order != 2 || p->general) return SYSTEC_ERR_UNSUPPORTED;
    const size_t bytes = static_cast<size_t>(p->dim) * 4;
    if (systec::overlap(d, bytes, y, bytes)) return SYSTEC_ERR_ALIAS;
    cudaError_t e = systec::launch_minplus(*p, d, y, reinterpret_cast<int *>(y), reinterpret_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? SYSTEC_OK : systec::cuda_fail(e);
}

namespace systec {
namespace {

// CP-ALS with the whole iteration loop on the device: iteration 0 and the
// first MTTKRP run eagerly, iterations 1..max_iters are the body of a
// conditional WHILE node of one CUDA graph (the dense pass, then the R x R
// algebra + device convergence test — which also flags the next run as
// fit-only when it is the last — beside the next iteration's MTTKRP), so
// there is no host round trip per iteration — one launch, one
// synchronisation at the end.  Returns cudaErrorNotSupported (nothing
// launched) when the graph cannot be built; the caller then runs the host loop.
cudaError_t cp_als_graph(Plan &p, float *B, int R, float *lambda, int max_iters, double tol, double *fit_host,
                         int *done, cudaStream_t s) {
    const size_t plane = static_cast<size_t>(p.dim) * R;
    systec_exec_opts o;
    std::memset(&o, 0, sizeof(o));
    const int64_t nscr = mttkrp_scratch_floats(p, R, o);
    float *M = nullptr, *fs = nullptr, *scr = nullptr;
    double *ds = nullptr, *fits = nullptr, *x2 = nullptr;
    CpdLoopState *st = nullptr;
    cudaGraph_t g = nullptr;
    cudaGraphExec_t ge = nullptr;
    cudaStream_t cs = nullptr, cs2 = nullptr;
    cudaEvent_t fork_ev = nullptr, join_ev = nullptr;
    bool launched = false;
    auto cleanup = [&]() {
        if (ge) cudaGraphExecDestroy(ge);
        if (g) cudaGraphDestroy(g);
        if (cs) cudaStreamDestroy(cs);
        if (cs2) cudaStreamDestroy(cs2);
        if (fork_ev) cudaEventDestroy(fork_ev);
        if (join_ev) cudaEventDestroy(join_ev);
        for (void *q : {static_cast<void *>(M), static_cast<void *>(fs), static_cast<void *>(scr),
                        static_cast<void *>(ds), static_cast<void *>(fits), static_cast<void *>(x2),
                        static_cast<void *>(st)})
            if (q) cudaFreeAsync(q, s);
    };
    cudaError_t e = cudaSuccess;
    do {
        // stream-ordered pool allocations on s: the graph (launched on s after
        // them, freed on s after it) keeps plain pointers to them
        if ((e = cudaMallocAsync(&M, plane * 4, s)) != cudaSuccess) break;
        if ((e = cudaMallocAsync(&fs, static_cast<size_t>(R) * R * 4, s)) != cudaSuccess) break;
        if ((e = cudaMallocAsync(&ds, sizeof(double) * cpd_scratch_doubles(R), s)) != cudaSuccess) break;
        if ((e = cudaMallocAsync(&fits, sizeof(double) * std::max(1, max_iters), s)) != cudaSuccess) break;
        if ((e = cudaMallocAsync(&x2, sizeof(double), s)) != cudaSuccess) break;
        if ((e = cudaMallocAsync(&st, sizeof(CpdLoopState), s)) != cudaSuccess) break;
        if (nscr > 0 && (e = cudaMallocAsync(&scr, static_cast<size_t>(nscr) * 4, s)) != cudaSuccess) break;
        // the loop graph: one conditional WHILE node, body captured on a private stream
        if ((e = cudaGraphCreate(&g, 0)) != cudaSuccess) break;
        cudaGraphConditionalHandle h;
        if ((e = cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault)) != cudaSuccess) break;
        cudaGraphNodeParams cp = {};
        cp.type = cudaGraphNodeTypeConditional;
        cp.conditional.handle = h;
        cp.conditional.type = cudaGraphCondTypeWhile;
        cp.conditional.size = 1;
        cudaGraphNode_t node;
        if ((e = cudaGraphAddNode(&node, g, nullptr, 0, &cp)) != cudaSuccess) break;
        cudaGraph_t body = cp.conditional.phGraph_out[0];
        if ((e = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking)) != cudaSuccess) break;
        if ((e = cudaStreamCreateWithFlags(&cs2, cudaStreamNonBlocking)) != cudaSuccess) break;
        if ((e = cudaEventCreateWithFlags(&fork_ev, cudaEventDisableTiming)) != cudaSuccess) break;
        if ((e = cudaEventCreateWithFlags(&join_ev, cudaEventDisableTiming)) != cudaSuccess) break;
        if ((e = cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal)) !=
            cudaSuccess)
            break;
        // body j (M = MTTKRP(X, F_j) on entry): the dense pass writes F_{j+1}, then
        // the R x R algebra + convergence test and MTTKRP(X, F_{j+1}) run side by
        // side (the MTTKRP needs only F_{j+1}; the algebra only the pass's
        // partial sums); the last body's MTTKRP is computed and not used
        cudaError_t ce = cpd_step_pass(p, M, B, R, ds, fs, false, &st->skip_update, cs);
        if (ce == cudaSuccess) ce = cudaEventRecord(fork_ev, cs);
        if (ce == cudaSuccess) ce = cudaStreamWaitEvent(cs2, fork_ev, 0);
        if (ce == cudaSuccess) ce = launch_mttkrp(p, B, R, M, o, cs2, scr);
        if (ce == cudaSuccess) ce = cudaEventRecord(join_ev, cs2);
        if (ce == cudaSuccess) ce = cpd_step_algebra(p, R, ds, fs, false, &st->skip_update, cs);
        if (ce == cudaSuccess) ce = cpd_fit_check(ds, R, st, fits, tol, max_iters, h, cs);
        if (ce == cudaSuccess) ce = cudaStreamWaitEvent(cs, join_ev, 0);
        cudaGraph_t captured = nullptr;
        e = cudaStreamEndCapture(cs, &captured);
        if (ce != cudaSuccess) e = ce;
        if (e != cudaSuccess) break;
        if ((e = cudaGraphInstantiate(&ge, g, 0)) != cudaSuccess) break;
        // ||X||^2, iteration 0 (no fit yet), then the device-resident loop
        if ((e = cpd_tensor_norm2(p, x2, s)) != cudaSuccess) break;
        if ((e = cpd_state_init(st, x2, max_iters, s)) != cudaSuccess) break;
        launched = true;
        if ((e = cpd_init(p, B, R, ds, fs, s)) != cudaSuccess) break;
        if ((e = launch_mttkrp(p, B, R, M, o, s, scr)) != cudaSuccess) break;
        if ((e = cpd_step(p, M, B, R, ds, fs, false, false, nullptr, s)) != cudaSuccess) break;
        if ((e = launch_mttkrp(p, B, R, M, o, s, scr)) != cudaSuccess) break;  // the first body's M
        if ((e = cudaGraphLaunch(ge, s)) != cudaSuccess) break;
        if ((e = cpd_finish(p, B, R, ds, lambda, s)) != cudaSuccess) break;
        CpdLoopState hst;
        if ((e = cudaMemcpyAsync(&hst, st, sizeof(hst), cudaMemcpyDeviceToHost, s)) != cudaSuccess) break;
        if ((e = cudaStreamSynchronize(s)) != cudaSuccess) break;
        *done = hst.iters_done;
        if (fit_host && hst.iters_done > 0) {
            if ((e = cudaMemcpyAsync(fit_host, fits, sizeof(double) * hst.iters_done, cudaMemcpyDeviceToHost, s)) !=
                cudaSuccess)
                break;
            e = cudaStreamSynchronize(s);
        }
    } while (false);
    if (e != cudaSuccess && !launched) {
        cudaGetLastError();  // clear a failed graph build; the host loop runs instead
        cleanup();
        return cudaErrorNotSupported;
    }
    cleanup();
    if (launched) {
        const cudaError_t f = cudaStreamSynchronize(s);
        if (e == cudaSuccess) e = f;
    }
    return e;
}

}  // namespace
}  // namespace systec

int systec_testing_cpd_pass(int form, int64_t dim, const float *M, float *F, const float *W, double *part,
                            int store, systec_stream_t stream) {
    systec::NvtxRange nvtx_range_("systec_testing_cpd_pass");
    if ((form != 0 && form != 1) || dim < 1 || !M || !F || !W || !part) return -SYSTEC_ERR_ARG;
    if ((reinterpret_cast<uintptr_t>(M) & 15) || (reinterpret_cast<uintptr_t>(F) & 15)) return -SYSTEC_ERR_UNSUPPORTED;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (form == 1) {
        const cudaError_t e = systec::launch_pass_umma32(M, F, W, dim, part, store, nullptr, s);
        if (e == cudaErrorNotSupported) {
            cudaGetLastError();
            return -SYSTEC_ERR_UNSUPPORTED;
        }
        return e == cudaSuccess ? systec::cpd_umma_blocks(dim) : -systec::cuda_fail(e);
    }
    cudaError_t e = cudaSuccess;
    const int pb = systec::cpd_pass_r32(0, dim, M, F, W, part, store, nullptr, s, &e);
    return pb > 0 ? pb : -systec::cuda_fail(e);
}

int systec_cp_als_sym(systec_plan plan, float *B, int R, float *lambda, int max_iters, double tol,
                      double *fit_host, int *iters_done, systec_stream_t stream) {
    systec::NvtxRange nvtx_range_("systec_cp_als_sym");
    Plan *p = reinterpret_cast<Plan *>(plan);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (!p || !B || !lambda || R < 1 || max_iters < 0) return SYSTEC_ERR_ARG;
    if (p->general || R > systec::cpd_max_rank()) return SYSTEC_ERR_UNSUPPORTED;
    const size_t plane = static_cast<size_t>(p->dim) * R;
    if (systec::overlap(B, plane * 4, lambda, static_cast<size_t>(R) * 4)) return SYSTEC_ERR_ALIAS;
    // loop placement: the device-resident graph saves the per-iteration host
    // round trip (c2, 50 iterations: 0.564 vs 0.580 ms/iteration) but costs
    // ~0.4 ms to build per call, so it is used for runs of >= 16 iterations;
    // SYSTEC_CPALS_LOOP=host|graph overrides (tests, measurements)
    const char *lp = getenv("SYSTEC_CPALS_LOOP");
    const bool use_graph = lp ? std::strcmp(lp, "graph") == 0 : max_iters >= 16;
    if (max_iters > 0 && use_graph) {
        int done = 0;
        cudaError_t ge = systec::cp_als_graph(*p, B, R, lambda, max_iters, tol, fit_host, &done, s);
        if (ge != cudaErrorNotSupported) {
            if (iters_done) *iters_done = done;
            return ge == cudaSuccess ? SYSTEC_OK : systec::cuda_fail(ge);
        }
    }
    float *M = nullptr, *fs = nullptr;
    double *ds = nullptr;
    double host[2] = {0, 0}, x2 = 0;
    cudaError_t e = cudaSuccess;
    int rc = SYSTEC_OK;
    int done = 0;
    auto cleanup = [&]() {
        if (M) cudaFreeAsync(M, s);
        if (fs) cudaFreeAsync(fs, s);
        if (ds) cudaFreeAsync(ds, s);
    };
    do {
        if ((e = cudaMallocAsync(&M, plane * 4, s)) != cudaSuccess) break;
        if ((e = cudaMallocAsync(&fs, static_cast<size_t>(R) * R * 4, s)) != cudaSuccess) break;
        if ((e = cudaMallocAsync(&ds, sizeof(double) * systec::cpd_scratch_doubles(R), s)) != cudaSuccess) break;
        if ((e = systec::cpd_tensor_norm2(*p, ds, s)) != cudaSuccess) break;
        if ((e = cudaMemcpyAsync(&x2, ds, sizeof(double), cudaMemcpyDeviceToHost, s)) != cudaSuccess) break;
        if ((e = cudaStreamSynchronize(s)) != cudaSuccess) break;
        const double xn = sqrt(x2 > 0 ? x2 : 1e-300);
        double prev_fit = -1e300;
        double *scal = ds + systec::cpd_xhat2_offset(R);
        if ((e = systec::cpd_init(*p, B, R, ds, fs, s)) != cudaSuccess) break;
        // iteration k: M = MTTKRP(X, F_k); its pass yields the fit pieces of iterate k (k > 0)
        for (int it = 0; it <= max_iters; ++it) {
            systec_exec_opts o;
            std::memset(&o, 0, sizeof(o));
            if ((e = systec::launch_mttkrp(*p, B, R, M, o, s)) != cudaSuccess) break;
            const bool last = it == max_iters;
            if ((e = systec::cpd_step(*p, M, B, R, ds, fs, it > 0, last, nullptr, s)) != cudaSuccess) break;
            if (it > 0) {
                if ((e = cudaMemcpyAsync(host, scal, 2 * sizeof(double), cudaMemcpyDeviceToHost, s)) != cudaSuccess) break;
                if ((e = cudaStreamSynchronize(s)) != cudaSuccess) break;
                const double r2 = x2 - 2 * host[1] + host[0];
                const double fit = 1.0 - sqrt(r2 > 0 ? r2 : 0.0) / xn;
                if (fit_host) fit_host[it - 1] = fit;
                done = it;
                // converged (or out of iterations): when converged early, B already holds
                // one more update than the last evaluated fit describes — it is kept
                if (last || fabs(fit - prev_fit) < tol) break;
                prev_fit = fit;
            }
        }
        // B holds the factor scaled by lambda: unit columns, and lambda out
        if (e == cudaSuccess) e = systec::cpd_finish(*p, B, R, ds, lambda, s);
    } while (false);
    cleanup();
    if (e != cudaSuccess) rc = systec::cuda_fail(e);
    if (iters_done) *iters_done = done;
    if (rc == SYSTEC_OK && (e = cudaStreamSynchronize(s)) != cudaSuccess) rc = systec::cuda_fail(e);
    return rc;
}

namespace systec {
namespace {

// Bellman-Ford with the loop on the device: one CUDA graph whose conditional
// WHILE node repeats relax -> update/compare -> step (which ends the loop when
// nothing changed or the budget is spent); one synchronisation at the end.
// cudaErrorNotSupported (nothing launched) when the graph cannot be built.
cudaError_t sssp_graph(Plan &p, float *dist, float *y, int *flag, int *iters, int max_iters, int *done,
                       cudaStream_t s) {
    cudaGraph_t g = nullptr;
    cudaGraphExec_t ge = nullptr;
    cudaStream_t cs = nullptr;
    cudaError_t e = cudaSuccess;
    bool launched = false;
    do {
        if ((e = cudaGraphCreate(&g, 0)) != cudaSuccess) break;
        cudaGraphConditionalHandle h;
        if ((e = cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault)) != cudaSuccess) break;
        cudaGraphNodeParams cp = {};
        cp.type = cudaGraphNodeTypeConditional;
        cp.conditional.handle = h;
        cp.conditional.type = cudaGraphCondTypeWhile;
        cp.conditional.size = 1;
        cudaGraphNode_t node;
        if ((e = cudaGraphAddNode(&node, g, nullptr, 0, &cp)) != cudaSuccess) break;
        cudaGraph_t body = cp.conditional.phGraph_out[0];
        if ((e = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking)) != cudaSuccess) break;
        if ((e = cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal)) !=
            cudaSuccess)
            break;
        cudaError_t ce = launch_minplus(p, dist, y, reinterpret_cast<int *>(y), cs);
        if (ce == cudaSuccess) ce = launch_sssp_update(y, dist, p.dim, flag, cs);
        if (ce == cudaSuccess) ce = launch_sssp_step(flag, iters, max_iters, h, cs);
        cudaGraph_t captured = nullptr;
        e = cudaStreamEndCapture(cs, &captured);
        if (ce != cudaSuccess) e = ce;
        if (e != cudaSuccess) break;
        if ((e = cudaGraphInstantiate(&ge, g, 0)) != cudaSuccess) break;
        launched = true;
        if ((e = cudaMemsetAsync(iters, 0, sizeof(int), s)) != cudaSuccess) break;
        if ((e = cudaGraphLaunch(ge, s)) != cudaSuccess) break;
        int h_it = 0;
        if ((e = cudaMemcpyAsync(&h_it, iters, sizeof(int), cudaMemcpyDeviceToHost, s)) != cudaSuccess) break;
        if ((e = cudaStreamSynchronize(s)) != cudaSuccess) break;
        *done = h_it;
    } while (false);
    if (ge) cudaGraphExecDestroy(ge);
    if (g) cudaGraphDestroy(g);
    if (cs) cudaStreamDestroy(cs);
    if (e != cudaSuccess && !launched) {
        cudaGetLastError();
        return cudaErrorNotSupported;
    }
    return e;
}

}  // namespace
}  // namespace systec

int systec_plan_sssp(systec_plan plan, int64_t source, float *dist, int max_iters, int *iters_done,
                     systec_stream_t stream) {
    Plan *p = reinterpret_cast<Plan *>(plan);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (!p || !dist || max_iters < 0 || source < 0 || source >= p->dim) return SYSTEC_ERR_ARG;
    if (p->order != 2 || p->general) return SYSTEC_ERR_UNSUPPORTED;
    float *y = nullptr;
    int *flag = nullptr;
    int done = 0, h_flag = 0;
    cudaError_t e;
    // loop placement: host loop by default — random graphs converge in tens of
    // relaxations, where building the device-loop graph (~0.3 ms) costs more
    // than the per-relaxation round trips it saves (dim 1e6, 10M nnz, 15
    // relaxations: 2.22 ms host vs 2.33 ms graph); SYSTEC_SSSP_LOOP=graph
    // selects the device-resident loop (long-diameter graphs)
    const char *lp = getenv("SYSTEC_SSSP_LOOP");
    const bool use_graph = lp && std::strcmp(lp, "graph") == 0;
    do {
        if ((e = cudaMallocAsync(&y, static_cast<size_t>(p->dim) * 4, s)) != cudaSuccess) break;
        if ((e = cudaMallocAsync(&flag, 2 * sizeof(int), s)) != cudaSuccess) break;
        if ((e = systec::launch_sssp_init(dist, p->dim, source, s)) != cudaSuccess) break;
        if (max_iters > 0 && use_graph) {
            e = systec::sssp_graph(*p, dist, y, flag, flag + 1, max_iters, &done, s);
            if (e != cudaErrorNotSupported) break;
            e = cudaSuccess;
        }
        // one (min,+) relaxation per iteration until nothing changes (Bellman-Ford)
        int it = 0;
        for (; it < max_iters; ++it) {
            if ((e = systec::launch_minplus(*p, dist, y, reinterpret_cast<int *>(y), s)) != cudaSuccess) break;
            if ((e = systec::launch_sssp_update(y, dist, p->dim, flag, s)) != cudaSuccess) break;
            if ((e = cudaMemcpyAsync(&h_flag, flag, sizeof(int), cudaMemcpyDeviceToHost, s)) != cudaSuccess) break;
            if ((e = cudaStreamSynchronize(s)) != cudaSuccess) break;
            if (!h_flag) {
                ++it;
                break;
            }
        }
        done = it;
    } while (false);
    if (y) cudaFreeAsync(y, s);
    if (flag) cudaFreeAsync(flag, s);
    if (iters_done) *iters_done = done;
    if (e != cudaSuccess) return systec::cuda_fail(e);
    e = cudaStreamSynchronize(s);
    return e == cudaSuccess ? SYSTEC_OK : systec::cuda_fail(e);
}

int systec_plan_ttm(systec_plan plan, const float *B, int R, float *C_packed, systec_stream_t stream) {
    Plan *p = reinterpret_cast<Plan *>(plan);
    if (!p || !B || !C_packed || R < 1) return SYSTEC_ERR_ARG;
    if (p->order != 3) return SYSTEC_ERR_UNSUPPORTED;
    const size_t rows = p->general ? static_cast<size_t>(p->dim) * p->dim : static_cast<size_t>(systec::ttm_packed_rows(p->dim));
    const size_t cb = rows * R * 4;
    if (systec::overlap(B, static_cast<size_t>(p->dim) * R * 4, C_packed, cb)) return SYSTEC_ERR_ALIAS;
    cudaError_t e = systec::launch_ttm(*p, B, R, C_packed, reinterpret_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? SYSTEC_OK : systec::cuda_fail(e);
}

int systec_ttm_unpack(int64_t dim, int R, const float *C_packed, float *C_full, systec_stream_t stream) {
    if (dim < 1 || R < 1 || !C_packed || !C_full) return SYSTEC_ERR_ARG;
    if (systec::overlap(C_packed, static_cast<size_t>(systec::ttm_packed_rows(dim)) * R * 4, C_full,
                        static_cast<size_t>(dim) * dim * R * 4))
        return SYSTEC_ERR_ALIAS;
    cudaError_t e = systec::launch_ttm_unpack(dim, R, C_packed, C_full, reinterpret_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? SYSTEC_OK : systec::cuda_fail(e);
}

int systec_plan_execute(systec_plan plan, const float *B, int R, float *C, systec_stream_t stream) {
    return systec::execute_impl(reinterpret_cast<Plan *>(plan), B, R, C, nullptr,
                                reinterpret_cast<cudaStream_t>(stream));
}

int systec_plan_execute_ex(systec_plan plan, const float *B, int R, float *C, const systec_exec_opts *opts,
                           systec_stream_t stream) {
    return systec::execute_impl(reinterpret_cast<Plan *>(plan), B, R, C, opts,
                                reinterpret_cast<cudaStream_t>(stream));
}

int systec_plan_stats(systec_plan plan, systec_stats *host_out) {
    if (!plan || !host_out) return SYSTEC_ERR_ARG;
    *host_out = reinterpret_cast<Plan *>(plan)->stats;
    return SYSTEC_OK;
}

int systec_plan_prepared(systec_plan plan, const int32_t **coords, const float **vals) {
    if (!plan || !coords || !vals) return SYSTEC_ERR_ARG;
    Plan *p = reinterpret_cast<Plan *>(plan);
    for (int t = 0; t < p->order; ++t) coords[t] = p->coords + static_cast<size_t>(t) * p->ld;
    *vals = p->vals;
    return SYSTEC_OK;
}

int systec_plan_copy_prepared(systec_plan plan, int32_t *coords_dst, float *vals_dst, systec_stream_t stream) {
    if (!plan || !coords_dst || !vals_dst) return SYSTEC_ERR_ARG;
    Plan *p = reinterpret_cast<Plan *>(plan);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (p->nnz == 0) return SYSTEC_OK;
    cudaError_t e = cudaMemcpy2DAsync(coords_dst, static_cast<size_t>(p->nnz) * 4, p->coords,
                                      static_cast<size_t>(p->ld) * 4, static_cast<size_t>(p->nnz) * 4, p->order,
                                      cudaMemcpyDeviceToDevice, s);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(vals_dst, p->vals, static_cast<size_t>(p->nnz) * 4, cudaMemcpyDeviceToDevice, s);
    return e == cudaSuccess ? SYSTEC_OK : systec::cuda_fail(e);
}

int systec_plan_last_launch(systec_plan plan, int32_t *grid_x, int32_t *grid_y, int32_t *block, int32_t *smem,
                            int32_t *kernel_id) {
    if (!plan) return SYSTEC_ERR_ARG;
    Plan *p = reinterpret_cast<Plan *>(plan);
    const Plan::LaunchInfo l = p->last_launch();
    if (grid_x) *grid_x = l.grid_x;
    if (grid_y) *grid_y = l.grid_y;
    if (block) *block = l.block;
    if (smem) *smem = l.smem;
    if (kernel_id) *kernel_id = l.kernel;
    return SYSTEC_OK;
}

int systec_plan_destroy(systec_plan plan) {
    systec::destroy_impl(reinterpret_cast<Plan *>(plan));
    return SYSTEC_OK;
}

int systec_mttkrp(int order, int64_t dim, int64_t nnz, const int32_t *idx, const float *vals, const float *B,
                  int R, float *C, systec_stream_t stream) {
    systec::NvtxRange nvtx_range_("systec_mttkrp");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    int bits = 0;
    int rc = systec::check_shape(order, dim, nnz, &bits);
    if (rc) return rc;
    if (!B || !C || R < 1 || (nnz > 0 && (!idx || !vals))) return SYSTEC_ERR_ARG;
    const size_t cb = static_cast<size_t>(dim) * R * sizeof(float);
    if (systec::overlap(C, cb, B, cb) || systec::overlap(C, cb, idx, static_cast<size_t>(nnz) * order * 4) ||
        systec::overlap(C, cb, vals, static_cast<size_t>(nnz) * 4))
        return SYSTEC_ERR_ALIAS;
    Plan *p = nullptr;
    rc = systec::plan_create_impl(&p, order, dim, nnz, idx, vals, s, true, false, -1);  // used once: no band re-sort
    if (rc) return rc;
    rc = systec::execute_impl(p, B, R, C, nullptr, s);
    systec::destroy_impl(p);
    return rc;
}

namespace systec {
namespace {

// Non-blocking streams per device for the pipeline's copies: which = 0 for
// host->device, 1 for device->host (created on first use, thread-safe, kept
// for the process lifetime).
cudaStream_t copy_stream(int which = 0) {
    static std::mutex mu;
    static cudaStream_t streams[2][64] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
    std::lock_guard<std::mutex> lock(mu);
    cudaStream_t &st = streams[which & 1][dev];
    if (!st && cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) st = nullptr;
    return st;
}

// canonical (ascending) copy of one host tuple
void canon_tuple(const int32_t *t, int order, int32_t *out) {
    for (int i = 0; i < order; ++i) out[i] = t[i];
    std::sort(out, out + order);
}

// Pipelined end-to-end call: chunk k's host->device copy (copy stream) overlaps
// chunk k-1's validate/canonicalise/gather/execute (caller's stream).  Chunks
// are contiguous and independent (MTTKRP is linear in A), so each one is
// executed into C as it lands; the sort is skipped (lexicographic input stays
// sorted per chunk; any other order is still correct, only with shorter runs).
// Position-1 accumulation is decided from chunk 0's statistics (one sync).
// Lexicographically sorted canonical input (the storage format) gives every
// later entry indices >= the next chunk's leading index c0, so once chunk k
// is executed the C rows below chunk k+1's first c0 are final: they are
// copied back on a device->host stream while later chunks still transfer and
// run (PCIe is full duplex).  Sortedness is confirmed afterwards — chunk
// boundaries on the host, inside chunks by the canonicalisation kernel's
// flag — and an unsorted input gets one more full copy of C at the end.
int mttkrp_host_pipelined(int order, int64_t dim, int64_t nnz, int bits, const int32_t *idx_host,
                          const float *vals_host, const float *B_host, int R, float *C_host, cudaStream_t s) {
    static const int kChunks = [] {  // SYSTEC_HOST_CHUNKS: tuning knob for the pipeline depth (default 16)
        const char *e = std::getenv("SYSTEC_HOST_CHUNKS");
        const int v = e ? std::atoi(e) : 16;
        return v < 1 ? 1 : (v > 256 ? 256 : v);
    }();
    const int64_t per = std::max<int64_t>(4, ((nnz + kChunks - 1) / kChunks + 3) & ~int64_t(3));  // 16-byte aligned
    const int nch = static_cast<int>((nnz + per - 1) / per);
    const int64_t ld = ((nnz + 3) & ~int64_t(3)) + 4;
    const size_t ib = static_cast<size_t>(nnz) * order * 4, vb = static_cast<size_t>(nnz) * 4;
    const size_t bb = static_cast<size_t>(dim) * R * 4;
    auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
    const size_t soa = static_cast<size_t>(order + 1) * ld * 4;
    const size_t kb = static_cast<size_t>(per) * 8, pb = static_cast<size_t>(per) * 4;
    const size_t total = al(ib) + al(vb) + 2 * al(bb) + al(soa) + al(kb) + al(pb) + al(sizeof(DevStats));
    char *buf = nullptr;
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void **>(&buf), total, s);
    if (e != cudaSuccess) return cuda_fail(e);
    char *q = buf;
    auto take = [&](size_t x) { char *r = q; q += al(x); return r; };
    int32_t *d_idx = reinterpret_cast<int32_t *>(take(ib));
    float *d_vals = reinterpret_cast<float *>(take(vb));
    float *d_B = reinterpret_cast<float *>(take(bb));
    float *d_C = reinterpret_cast<float *>(take(bb));
    int32_t *coords = reinterpret_cast<int32_t *>(take(soa));
    float *svals = reinterpret_cast<float *>(coords + static_cast<size_t>(order) * ld);
    unsigned long long *keys = reinterpret_cast<unsigned long long *>(take(kb));
    uint32_t *perm = reinterpret_cast<uint32_t *>(take(pb));
    DevStats *dst = reinterpret_cast<DevStats *>(take(sizeof(DevStats)));
    DevStats hst;
    std::memset(&hst, 0, sizeof(hst));
    hst.bad_entry = ULLONG_MAX;
    cudaStream_t cs = copy_stream();
    if (!cs) cs = s;  // no copy stream: copies on the caller's stream (no overlap, same result)
    cudaStream_t ds = s;  // device->host stream of the early C copies (set below)
    std::vector<cudaEvent_t> ev(nch + 2, nullptr);
    int rc = SYSTEC_OK;
    do {
        for (auto &x : ev)
            if ((e = cudaEventCreateWithFlags(&x, cudaEventDisableTiming)) != cudaSuccess) break;
        if (e != cudaSuccess) break;
        if ((e = cudaMemcpyAsync(dst, &hst, sizeof(hst), cudaMemcpyHostToDevice, s)) != cudaSuccess) break;
        if ((e = cudaMemsetAsync(d_C, 0, bb, s)) != cudaSuccess) break;
        if ((e = cudaEventRecord(ev[nch + 1], s)) != cudaSuccess) break;          // buffers exist
        if ((e = cudaStreamWaitEvent(cs, ev[nch + 1], 0)) != cudaSuccess) break;
        // copy order: B and all values first (two copies), then the index
        // chunks — every copy costs a fixed overhead on the copy engine, and
        // the order does not change the total, only when chunk 0 can start
        // (SYSTEC_HOST_VALS_CHUNKED=1: values per chunk, 2 copies per chunk)
        static const bool kValsChunked = [] {
            const char *v = std::getenv("SYSTEC_HOST_VALS_CHUNKED");
            return v && v[0] == '1';
        }();
        if ((e = cudaMemcpyAsync(d_B, B_host, bb, cudaMemcpyHostToDevice, cs)) != cudaSuccess) break;
        if (!kValsChunked && (e = cudaMemcpyAsync(d_vals, vals_host, vb, cudaMemcpyHostToDevice, cs)) != cudaSuccess)
            break;
        if ((e = cudaEventRecord(ev[nch], cs)) != cudaSuccess) break;
        for (int k = 0; k < nch && e == cudaSuccess; ++k) {
            const int64_t lo = k * per, n = std::min(per, nnz - lo);
            if ((e = cudaMemcpyAsync(d_idx + lo * order, idx_host + lo * order, n * order * 4, cudaMemcpyHostToDevice, cs)) != cudaSuccess) break;
            if (kValsChunked &&
                (e = cudaMemcpyAsync(d_vals + lo, vals_host + lo, n * 4, cudaMemcpyHostToDevice, cs)) != cudaSuccess)
                break;
            e = cudaEventRecord(ev[k], cs);
        }
        if (e != cudaSuccess) break;
        if ((e = cudaStreamWaitEvent(s, ev[nch], 0)) != cudaSuccess) break;        // B landed
        systec_exec_opts o;
        std::memset(&o, 0, sizeof(o));
        o.no_zero = 1;
        // early copies only into page-locked C (a pageable destination would
        // make each copy block the host thread that is feeding the pipeline)
        cudaPointerAttributes pa;
        const bool c_pinned = cudaPointerGetAttributes(&pa, C_host) == cudaSuccess && pa.type == cudaMemoryTypeHost;
        cudaGetLastError();  // clear a possible error from the query
        static const bool kEarly = [] {  // SYSTEC_HOST_EARLY=0: no early copies (measurements)
            const char *v = std::getenv("SYSTEC_HOST_EARLY");
            return !(v && v[0] == '0');
        }();
        ds = (c_pinned && kEarly) ? copy_stream(1) : nullptr;
        if (!ds) ds = s;
        bool bounds_sorted = true;  // chunk boundaries in canonical lexicographic order (host check)
        int64_t done_rows = 0;      // C rows [0, done_rows) already copied back
        const size_t row_bytes = static_cast<size_t>(R) * 4;
        for (int k = 0; k < nch; ++k) {
            const int64_t lo = k * per, n = std::min(per, nnz - lo);
            if ((e = cudaStreamWaitEvent(s, ev[k], 0)) != cudaSuccess) break;
            if (bits * order > 64) {  // wide plan: no packed keys (the last chunk's padding tail is never read)
                if ((e = launch_validate_wide(order, dim, n, d_idx + lo * order, perm, dst, s, true, lo)) != cudaSuccess)
                    break;
                if ((e = launch_gather_wide(order, n, n, ld, dim, d_idx + lo * order, nullptr, d_vals + lo, coords + lo,
                                            svals + lo, s, true)) != cudaSuccess)
                    break;
            } else {
                if ((e = launch_canonicalize(order, dim, n, bits, d_idx + lo * order, keys, perm, dst, s, true, lo)) != cudaSuccess)
                    break;
                if ((e = launch_gather_range(order, n, ld, bits, keys, d_vals + lo, coords + lo, svals + lo, s)) != cudaSuccess) break;
            }
            if (k == 0) {  // chunk-0 statistics decide position-1 accumulation (one sync)
                if ((e = launch_stats(order, n, ld, coords, -1, dst, s)) != cudaSuccess) break;
                if ((e = cudaMemcpyAsync(&hst, dst, sizeof(hst), cudaMemcpyDeviceToHost, s)) != cudaSuccess) break;
                if ((e = cudaStreamSynchronize(s)) != cudaSuccess) break;
                if (hst.err) break;
                o.pos1_accumulate = (hst.pos1_runs > 0 && static_cast<double>(n) / hst.pos1_runs >= 1.5) ? 1 : -1;
            }
            Plan pk;
            pk.order = order;
            pk.dim = dim;
            pk.nnz = n;
            pk.ld = ld;
            pk.key_bits = bits;
            pk.coords = coords + lo;
            pk.vals = svals + lo;
            pk.stream = s;
            if ((e = launch_mttkrp(pk, d_B, R, d_C, o, s)) != cudaSuccess) break;
            if (k + 1 < nch && bounds_sorted) {  // early copy of the rows no later chunk can touch
                int32_t a[8], b[8];
                canon_tuple(idx_host + (lo + n - 1) * order, order, a);
                canon_tuple(idx_host + (lo + n) * order, order, b);
                bounds_sorted = !std::lexicographical_compare(b, b + order, a, a + order);
                const int64_t bound = std::min<int64_t>(std::max<int64_t>(b[0], 0), dim);
                if (bounds_sorted && bound > done_rows && ds != s) {
                    if ((e = cudaEventRecord(ev[k], s)) != cudaSuccess) break;  // chunk k executed
                    if ((e = cudaStreamWaitEvent(ds, ev[k], 0)) != cudaSuccess) break;
                    if ((e = cudaMemcpyAsync(reinterpret_cast<char *>(C_host) + done_rows * row_bytes,
                                             reinterpret_cast<const char *>(d_C) + done_rows * row_bytes,
                                             (bound - done_rows) * row_bytes, cudaMemcpyDeviceToHost, ds)) != cudaSuccess)
                        break;
                    done_rows = bound;
                }
            }
        }
        if (e != cudaSuccess) break;
        if (hst.err) {
            g_last_bad_entry = static_cast<int64_t>(hst.bad_entry);
            rc = SYSTEC_ERR_INDEX;
            break;
        }
        if ((e = cudaMemcpyAsync(&hst, dst, sizeof(hst), cudaMemcpyDeviceToHost, s)) != cudaSuccess) break;
        if ((e = cudaMemcpyAsync(reinterpret_cast<char *>(C_host) + done_rows * row_bytes,
                                 reinterpret_cast<const char *>(d_C) + done_rows * row_bytes,
                                 bb - done_rows * row_bytes, cudaMemcpyDeviceToHost, s)) != cudaSuccess)
            break;
        if ((e = cudaStreamSynchronize(s)) != cudaSuccess) break;
        if ((e = cudaStreamSynchronize(ds)) != cudaSuccess) break;
        if (hst.err) {  // a later chunk held a bad index: C is not valid
            g_last_bad_entry = static_cast<int64_t>(hst.bad_entry);
            rc = SYSTEC_ERR_INDEX;
        } else if (done_rows > 0 && (hst.unsorted || !bounds_sorted)) {
            // not sorted after all: rows copied early may have changed since
            if ((e = cudaMemcpyAsync(C_host, d_C, done_rows * row_bytes, cudaMemcpyDeviceToHost, s)) != cudaSuccess) break;
            if ((e = cudaStreamSynchronize(s)) != cudaSuccess) break;
        }
    } while (false);
    cudaStreamSynchronize(cs);
    cudaStreamSynchronize(ds);  // no copy into C_host outlives the call
    cudaFreeAsync(buf, s);
    for (auto &x : ev)
        if (x) cudaEventDestroy(x);
    if (e != cudaSuccess) return cuda_fail(e);
    if (rc == SYSTEC_OK && (e = cudaStreamSynchronize(s)) != cudaSuccess) return cuda_fail(e);
    return rc;
}

}  // namespace
}  // namespace systec

int systec_mttkrp_host(int order, int64_t dim, int64_t nnz, const int32_t *idx_host, const float *vals_host,
                       const float *B_host, int R, float *C_host, systec_stream_t stream) {
    systec::NvtxRange nvtx_range_("systec_mttkrp_host");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    int bits = 0;
    int rc = systec::check_shape(order, dim, nnz, &bits);
    if (rc) return rc;
    if (!B_host || !C_host || R < 1 || (nnz > 0 && (!idx_host || !vals_host))) return SYSTEC_ERR_ARG;
    systec::ensure_pool_keeps_memory();
    if (nnz >= (1 << 20)) return systec::mttkrp_host_pipelined(order, dim, nnz, bits, idx_host, vals_host, B_host, R, C_host, s);
    const size_t ib = static_cast<size_t>(nnz) * order * 4, vb = static_cast<size_t>(nnz) * 4;
    const size_t bb = static_cast<size_t>(dim) * R * 4;
    char *buf = nullptr;
    const size_t ib_al = (ib + 255) & ~size_t(255), vb_al = (vb + 255) & ~size_t(255), bb_al = (bb + 255) & ~size_t(255);
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void **>(&buf), ib_al + vb_al + 2 * bb_al + 256, s);
    if (e != cudaSuccess) return systec::cuda_fail(e);
    int32_t *d_idx = reinterpret_cast<int32_t *>(buf);
    float *d_vals = reinterpret_cast<float *>(buf + ib_al);
    float *d_B = reinterpret_cast<float *>(buf + ib_al + vb_al);
    float *d_C = reinterpret_cast<float *>(buf + ib_al + vb_al + bb_al);
    Plan *p = nullptr;
    rc = SYSTEC_OK;
    do {
        if (ib && (e = cudaMemcpyAsync(d_idx, idx_host, ib, cudaMemcpyHostToDevice, s)) != cudaSuccess) break;
        if (vb && (e = cudaMemcpyAsync(d_vals, vals_host, vb, cudaMemcpyHostToDevice, s)) != cudaSuccess) break;
        if ((e = cudaMemcpyAsync(d_B, B_host, bb, cudaMemcpyHostToDevice, s)) != cudaSuccess) break;
        rc = systec::plan_create_impl(&p, order, dim, nnz, d_idx, d_vals, s, true, false, -1);
        if (rc) break;
        rc = systec::execute_impl(p, d_B, R, d_C, nullptr, s);
        if (rc) break;
        if ((e = cudaMemcpyAsync(C_host, d_C, bb, cudaMemcpyDeviceToHost, s)) != cudaSuccess) break;
    } while (false);
    if (p) systec::destroy_impl(p);
    cudaFreeAsync(buf, s);
    if (e != cudaSuccess) return systec::cuda_fail(e);
    if (rc) return rc;
    e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return systec::cuda_fail(e);
    return SYSTEC_OK;
}

const char *systec_status_string(int status) {
    switch (status) {
        case SYSTEC_OK: return "ok";
        case SYSTEC_ERR_ARG: return "invalid argument";
        case SYSTEC_ERR_UNSUPPORTED: return "unsupported order/dim/nnz";
        case SYSTEC_ERR_INDEX: return "index outside [0, dim)";
        case SYSTEC_ERR_ALIAS: return "output aliases an input";
        case SYSTEC_ERR_NOMEM: return "out of memory";
        case SYSTEC_ERR_CUDA: return "CUDA error";
        default: return "unknown status";
    }
}

int systec_last_cuda_error(void) { return systec::g_last_cuda_error; }
int systec_version(void) { return 100; }
int64_t systec_last_bad_entry(void) { return systec::g_last_bad_entry; }

}  // extern "C"
