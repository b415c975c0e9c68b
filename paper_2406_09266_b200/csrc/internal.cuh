// internal.cuh — plan object and launcher declarations shared by the .cu files
// of libsystec (not part of the public ABI; see include/systec.h).
#pragma once
#include <cstdint>
#include <mutex>
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include "../../include/systec.h"

namespace systec {

// NVTX range around an ABI call (prepare / execute / host call / CP-ALS):
// visible in Nsight timelines, a no-op without an attached tool
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange &) = delete;
    NvtxRange &operator=(const NvtxRange &) = delete;
};

// Prepared, canonicalised, lexicographically sorted structure-of-arrays stream.
struct Plan {
    int order = 0;
    int64_t dim = 0;
    int64_t nnz = 0;
    int64_t ld = 0;            // padded length of every array (multiple of 4, >= nnz)
    int key_bits = 0;
    int band_shift = -1;       // >= 0: entries grouped by band c_{n-1} >> band_shift, lexicographic within a band
    int32_t *coords = nullptr; // [order][ld] int32: c_t of entry e at coords[t*ld + e]
    float *vals = nullptr;     // [ld] fp32
    void *storage = nullptr;   // one allocation holding coords + vals
    bool pooled = false;       // storage from the stream-ordered pool (freed async)
    bool general = false;      // non-symmetric tensor: tuples kept as given, naive kernel
    cudaStream_t stream = nullptr;
    systec_stats stats{};
    // order-2 windowed kernel (sym2_window.cu): row pointer and the upper
    // triangle's column pointer, [dim + 1] each, in one allocation
    int32_t *win_rowptr = nullptr, *win_colptr = nullptr;
    int64_t win_bw = 0;
    int win_capp = 0;          // partition step; 0 = no windowed path
    int win_nblk = 0;
    // last launch (for reporting).  Concurrent executes of one plan may run
    // on several host threads: the record is written and read under a mutex,
    // so a reader sees one whole launch (the most recent to finish recording).
    struct LaunchInfo {
        int grid_x = 0, grid_y = 0, block = 0, smem = 0, kernel = -1;
    };
    mutable std::mutex last_mu;
    mutable LaunchInfo last;
    void record_launch(const LaunchInfo &l) const {
        std::lock_guard<std::mutex> g(last_mu);
        last = l;
    }
    LaunchInfo last_launch() const {
        std::lock_guard<std::mutex> g(last_mu);
        return last;
    }
};

// Device-side counters filled by the prepare kernels (all unsigned 64-bit).
struct DevStats {
    unsigned long long err;            // bit 0: index out of range
    unsigned long long unsorted;       // 1 if canonical keys are not non-decreasing
    unsigned long long bad_entry;      // min entry with a bad index (ULLONG_MAX if none)
    unsigned long long G;
    unsigned long long expanded;
    unsigned long long hist[16];
    unsigned long long lead_runs;
    unsigned long long max_lead_run;
    unsigned long long pos1_runs;
};

// prepare.cu
cudaError_t launch_canonicalize(int order, int64_t dim, int64_t nnz, int bits, const int32_t *idx,
                                unsigned long long *keys, uint32_t *perm, DevStats *st,
                                cudaStream_t s, bool canonicalise = true, int64_t e_offset = 0);
cudaError_t sort_keys(int64_t nnz, int end_bit, unsigned long long *keys_in, unsigned long long *keys_out,
                      uint32_t *perm_in, uint32_t *perm_out, cudaStream_t s);
cudaError_t launch_gather(int order, int64_t nnz, int64_t ld, int bits, const unsigned long long *keys,
                          const uint32_t *perm /* null = identity */, const float *vals_in,
                          int32_t *coords, float *vals_out, cudaStream_t s);
cudaError_t launch_stats(int order, int64_t nnz, int64_t ld, const int32_t *coords, int band_shift, DevStats *st,
                         cudaStream_t s);
cudaError_t launch_band_keys(int order, int64_t nnz, int64_t ld, const int32_t *coords, int band_shift,
                             uint16_t *band, uint32_t *perm, cudaStream_t s);
cudaError_t sort_band_keys(int64_t nnz, int band_bits, uint16_t *keys_in, uint16_t *keys_out, uint32_t *perm_in,
                           uint32_t *perm_out, cudaStream_t s);
cudaError_t launch_permute(int order, int64_t nnz, int64_t ld, const uint32_t *perm, const int32_t *cin,
                           const float *vin, int32_t *cout, float *vout, cudaStream_t s);
cudaError_t launch_gather_range(int order, int64_t n, int64_t ld, int bits, const unsigned long long *keys,
                                const float *vals_in, int32_t *coords, float *vals_out, cudaStream_t s);

// one pass for input already in storage order: SoA stream + validation + sortedness + statistics
cudaError_t launch_prepare_sorted(int order, int64_t dim, int64_t nnz, int64_t ld, const int32_t *idx,
                                  const float *vals_in, int32_t *coords, float *vals_out, DevStats *st,
                                  cudaStream_t s, bool canonicalise = true, int64_t e_offset = 0);
// wide plans (order * ceil(log2 dim) > 64): no packed keys
cudaError_t launch_validate_wide(int order, int64_t dim, int64_t nnz, const int32_t *idx, uint32_t *perm,
                                 DevStats *st, cudaStream_t s, bool canonicalise = true, int64_t e_offset = 0);
cudaError_t sort_wide(int order, int64_t dim, int64_t nnz, int bits, const int32_t *idx, unsigned long long *keys,
                      unsigned long long *keys2, uint32_t *perm, uint32_t *perm2, uint32_t **perm_out,
                      cudaStream_t s, bool canonicalise = true);
// span: entries written (ld for a whole plan incl. its zero padding, nnz for one chunk of the host pipeline)
cudaError_t launch_gather_wide(int order, int64_t nnz, int64_t span, int64_t ld, int64_t dim, const int32_t *idx,
                               const uint32_t *perm /* null = identity */, const float *vals_in, int32_t *coords,
                               float *vals_out, cudaStream_t s, bool canonicalise = true);

// expand.cu
cudaError_t expand_count(int order, int64_t dim, int64_t nnz, const int32_t *idx, unsigned long long *sizes,
                         unsigned long long *offsets, DevStats *st, cudaStream_t s);
cudaError_t expand_write(int order, int64_t nnz, const int32_t *idx, const float *vals,
                         const unsigned long long *offsets, int32_t *out_idx, float *out_vals, cudaStream_t s);

// minplus.cu — keys may alias y (in-place order-preserving integer keys)
cudaError_t launch_minplus(const Plan &p, const float *d, float *y, int *scratch_keys, cudaStream_t s);
cudaError_t launch_sssp_init(float *d, int64_t dim, int64_t source, cudaStream_t s);
// d = y where different, *changed = any difference (zeroes *changed first)
cudaError_t launch_sssp_update(const float *y, float *d, int64_t dim, int *changed, cudaStream_t s);
cudaError_t launch_sssp_step(const int *changed, int *iters, int max_iters, cudaGraphConditionalHandle h,
                             cudaStream_t s);

// cpd.cu
int cpd_max_rank();
int64_t cpd_scratch_doubles(int R);
int64_t cpd_xhat2_offset(int R);  // doubles into the scratch: {||Xhat||^2, <X,Xhat>}
cudaError_t cpd_tensor_norm2(const Plan &p, double *out, cudaStream_t s);
// before iteration 0: the Gram of the caller's factor (carried from then on in
// the scratch), lambda = 1, and the first pass's W
cudaError_t cpd_init(const Plan &p, const float *B, int R, double *dscratch, float *fscratch, cudaStream_t s);
// one iteration after its MTTKRP M = MTTKRP(X, F): the dense pass (G_M, dots
// M o F, and F = M W unless fit_only or *skip), then the R x R algebra (the
// fit of the current iterate when have_lam; the new lambda, G_B and the next
// W unless fit_only or *skip).  F is stored with column scale lambda.
cudaError_t cpd_step(const Plan &p, const float *M, float *F, int R, double *dscratch, float *fscratch,
                     bool have_lam, bool fit_only, const int *skip, cudaStream_t s);
// the R = 32 dense pass in one form (0: mma.sync, 1: tcgen05; cpd_umma.cu):
// part[blocks] = {M^T M, dots M o F}, F = M W when store; returns the blocks
// used, or -1 when the form cannot run (form 1: misaligned / no encoder)
int cpd_pass_r32(int form, int64_t dim, const float *M, float *F, const float *W, double *part, int store,
                 const int *skip, cudaStream_t s, cudaError_t *err);
cudaError_t launch_pass_umma32(const float *M, float *F, const float *W, int64_t dim, double *part, int store,
                               const int *skip, cudaStream_t s);
int cpd_umma_blocks(int64_t dim);
// cpd_step (have_lam) in two parts: the dense pass with its partial-sum
// reduction, then the R x R algebra (the device loop runs the next MTTKRP
// beside the algebra: it only needs the F the pass wrote)
cudaError_t cpd_step_pass(const Plan &p, const float *M, float *F, int R, double *dscratch, const float *fscratch,
                          bool fit_only, const int *skip, cudaStream_t s);
cudaError_t cpd_step_algebra(const Plan &p, int R, double *dscratch, float *fscratch, bool fit_only, const int *skip,
                             cudaStream_t s);
// after the last iteration: F /= lambda (unit columns), lam = lambda (fp32)
cudaError_t cpd_finish(const Plan &p, float *F, int R, const double *dscratch, float *lam, cudaStream_t s);
// device-resident CP-ALS loop (one conditional-WHILE graph): state + pieces
struct CpdLoopState {
    double x2;         // ||X||^2
    double prev_fit;
    int it;            // iterations evaluated
    int skip_update;   // 1 on the last iteration: fit only
    int iters_done;
    int pad;
};
cudaError_t cpd_state_init(CpdLoopState *st, const double *x2, int max_iters, cudaStream_t s);
cudaError_t cpd_fit_check(const double *dscratch, int R, CpdLoopState *st, double *fits, double tol, int max_iters,
                          cudaGraphConditionalHandle h, cudaStream_t s);

// ttm.cu
int64_t ttm_packed_rows(int64_t dim);
cudaError_t launch_ttm(const Plan &p, const float *B, int R, float *Cp, cudaStream_t s);
cudaError_t launch_ttm_unpack(int64_t dim, int R, const float *Cp, float *C, cudaStream_t s);

// sym2_window.cu
cudaError_t win_build(const Plan &p, int32_t *rowptr, int32_t *colptr, unsigned long long *bw_dev,
                      unsigned long long *maxcol_dev, cudaStream_t s);
int win_partition(int64_t dim, int64_t items, int64_t bw, int64_t maxcol, int *nblk);
// cudaErrorNotSupported: the plan has no windowed path for this R / layout (nothing launched)
cudaError_t launch_sym2_window(const Plan &p, const float *B, int R, float *C, bool accumulate, cudaStream_t s);

// mttkrp.cu
cudaError_t launch_mttkrp(const Plan &p, const float *B, int R, float *C, const systec_exec_opts &o,
                          cudaStream_t s, float *scratch = nullptr);
// floats of replica scratch launch_mttkrp needs for (plan, R, opts); 0 = none.
// Passing that much as `scratch` makes the launch allocation-free (graph bodies).
int64_t mttkrp_scratch_floats(const Plan &p, int R, const systec_exec_opts &o);

void set_last_cuda_error(cudaError_t e);

}  // namespace systec
