// microbench_passes.cu — would a second, differently sorted copy of the stream
// pay on c2?  The c2 kernel is bound by the SM->L2 request port, which the
// reductions' write payload dominates.  A pass over a copy
// sorted by the LAST index turns that position's reductions into register
// runs at the cost of re-gathering the other rows.  This measures the c2-shaped
// synthetic loops (random 128-B rows of 12.8 MB tables, no stream, no run
// logic): G gathers + D reductions per entry, per 10M entries.
//
//   nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -o tools/microbench_passes tools/microbench_passes.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); return 1; } } while (0)

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
    return x;
}

template <int G, int D>
__global__ void mix(const float *__restrict__ B, float *C, uint32_t rows, int iters, float *sink) {
    const int lane = threadIdx.x & 31, g = lane >> 3, j = lane & 7;
    const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    float4 keep = make_float4(0, 0, 0, 0);
    for (int it = 0; it < iters; ++it) {
        const uint32_t h = gw * 131071u + it * 4u + g;
        float4 p = make_float4(1, 1, 1, 1);
        uint32_t r[G > D ? G : D];
#pragma unroll
        for (int t = 0; t < (G > D ? G : D); ++t) r[t] = hash32(h ^ (0x9e3779b9u * (t + 1))) % rows;
#pragma unroll
        for (int t = 0; t < G; ++t) {
            const float4 b = __ldg(reinterpret_cast<const float4 *>(B + (size_t)r[t] * 32) + j);
            p.x *= b.x; p.y *= b.y; p.z *= b.z; p.w *= b.w;
        }
#pragma unroll
        for (int t = 0; t < D; ++t) {
            float *q = C + (size_t)r[t] * 32 + j * 4;
            asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(q), "f"(p.x), "f"(p.y), "f"(p.z), "f"(p.w) : "memory");
        }
        keep.x += p.x; keep.y += p.y; keep.z += p.z; keep.w += p.w;
    }
    if (keep.x + keep.y + keep.z + keep.w == 12345.f) *sink = keep.x;
}

// both passes of a split plan co-running in one launch: each warp-iteration
// takes its next entry group from one shared counter space; groups below
// `na` are pass A (3 gathers, 1 reduction: positions 0..n-2 of the canonical
// stream), the rest pass B (2 gathers: position n-1 along runs)
__global__ void mix_ab(const float *__restrict__ B, float *C, uint32_t rows, unsigned na, unsigned total,
                      unsigned *ctr, float *sink) {
    const int lane = threadIdx.x & 31, g = lane >> 3, j = lane & 7;
    float4 keep = make_float4(0, 0, 0, 0);
    while (true) {
        unsigned t = 0;
        if (lane == 0) t = atomicAdd(ctr, 1u);
        t = __shfl_sync(0xffffffffu, t, 0);
        if (t >= total) break;
        // 32 entries-iterations per taken unit (as a 132-entry chunk would be)
        for (int it = 0; it < 32; ++it) {
            const uint32_t h = t * 131u + it * 4u + g;
            const uint32_t r0 = hash32(h) % rows, r1 = hash32(h ^ 0x9e3779b9u) % rows, r2 = hash32(h ^ 0x85ebca6bu) % rows;
            const float4 a = __ldg(reinterpret_cast<const float4 *>(B + (size_t)r0 * 32) + j);
            const float4 b = __ldg(reinterpret_cast<const float4 *>(B + (size_t)r1 * 32) + j);
            float4 p = make_float4(a.x * b.x, a.y * b.y, a.z * b.z, a.w * b.w);
            if (t < na) {  // pass A: the c0 row is an L1 hit in the real kernel: 2 random gathers + 1 red
                float *q = C + (size_t)r2 * 32 + j * 4;
                asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(q), "f"(p.x), "f"(p.y), "f"(p.z), "f"(p.w) : "memory");
            }
            keep.x += p.x; keep.y += p.y; keep.z += p.z; keep.w += p.w;
        }
    }
    if (keep.x + keep.y + keep.z + keep.w == 12345.f) *sink = keep.x;
}

template <int G, int D>
int run(const char *name, const float *B, float *C, uint32_t rows, int sms, float *sink, bool first) {
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    const int iters = 128, blocks = sms * 8, threads = 256;
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        CK(cudaEventRecord(e0));
        mix<G, D><<<blocks, threads>>>(B, C, rows, iters, sink);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        best = ms < best ? ms : best;
    }
    const double entries = (double)blocks * threads / 8 * iters;
    printf("%s\"%s\": %.4f", first ? "" : ", ", name, best * 1e7 / entries);
    return 0;
}

int main() {
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const uint32_t rows = 100000;  // 12.8 MB tables: c2's B and C
    float *B, *C, *sink;
    CK(cudaMalloc(&B, (size_t)rows * 128));
    CK(cudaMalloc(&C, (size_t)rows * 128));
    CK(cudaMalloc(&sink, 4));
    CK(cudaMemset(B, 0, (size_t)rows * 128));
    CK(cudaMemset(C, 0, (size_t)rows * 128));
    printf("{\"unit\": \"ms per 10M entries\"");
    printf(", ");
    int rc = 0;
    rc |= run<3, 2>("g3_r2 (one pass, today)", B, C, rows, sms, sink, true);
    rc |= run<3, 1>("g3_r1 (pass A of two)", B, C, rows, sms, sink, false);
    rc |= run<2, 0>("g2_r0 (pass sorted by last index)", B, C, rows, sms, sink, false);
    rc |= run<2, 1>("g2_r1", B, C, rows, sms, sink, false);
    rc |= run<3, 0>("g3_r0", B, C, rows, sms, sink, false);
    rc |= run<2, 2>("g2_r2 (one pass, c0 row from L1)", B, C, rows, sms, sink, false);
    rc |= run<0, 1>("g0_r1", B, C, rows, sms, sink, false);
    rc |= run<0, 2>("g0_r2", B, C, rows, sms, sink, false);
    // split plan, both passes in one launch with one shared work counter:
    // 10M pass-A entries (g2_r1 with the c0 row from L1 modelled as a 3rd
    // gather) + 10M pass-B entries, vs the single pass (g2_r2 / g3_r2)
    {
        unsigned *ctr;
        CK(cudaMalloc(&ctr, 4));
        const unsigned per_unit = 32 * 4;  // entries per taken unit (4 groups x 32 iterations)
        const unsigned na = 10000000u / per_unit, total = 2 * na;
        cudaEvent_t e0, e1;
        CK(cudaEventCreate(&e0));
        CK(cudaEventCreate(&e1));
        float best = 1e30f;
        for (int r = 0; r < 5; ++r) {
            CK(cudaMemset(ctr, 0, 4));
            CK(cudaEventRecord(e0));
            mix_ab<<<sms * 8, 256>>>(B, C, rows, na, total, ctr, sink);
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            float ms;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            best = ms < best ? ms : best;
        }
        printf(", \"split_AB_one_launch (10M A g2_r1 + 10M B g2_r0)\": %.4f", best);
    }
    printf("}\n");
    return rc;
}
