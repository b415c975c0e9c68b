// microbench.cu — measures the bounds the symmetric MTTKRP actually runs into
// on this B200: HBM stream read, L2 random-row gather of
// B-like tables, vector red.global throughput into random C rows, and the
// same-row contention rate.  Prints one JSON object.
//
//   nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -o tools/microbench tools/microbench.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); return 1; } } while (0)

__global__ void stream_read(const float4 *__restrict__ a, size_t n4, float *sink) {
    float4 acc = make_float4(0, 0, 0, 0);
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
        float4 v = __ldg(a + i);
        acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    if (acc.x + acc.y + acc.z + acc.w == 12345.f) *sink = acc.x;
}

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
    return x;
}

// each group of 8 lanes gathers one 128-byte row (R = 32 floats) per iteration
__global__ void gather_rows(const float *__restrict__ B, uint32_t rows, int iters, float *sink) {
    const int lane = threadIdx.x & 31, g = lane >> 3, j = lane & 7;
    const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    float4 acc = make_float4(0, 0, 0, 0);
#pragma unroll 4
    for (int it = 0; it < iters; ++it) {
        const uint32_t r = hash32(gw * 131071u + it * 4u + g) % rows;
        float4 v = __ldg(reinterpret_cast<const float4 *>(B + (size_t)r * 32) + j);
        acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    if (acc.x + acc.y + acc.z + acc.w == 12345.f) *sink = acc.x;
}

__global__ void red_rows(float *C, uint32_t rows, int iters) {
    const int lane = threadIdx.x & 31, g = lane >> 3, j = lane & 7;
    const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const float4 v = make_float4(1.f, 1.f, 1.f, 1.f);
    for (int it = 0; it < iters; ++it) {
        const uint32_t r = hash32(gw * 131071u + it * 4u + g) % rows;
        float *p = C + (size_t)r * 32 + j * 4;
        asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
    }
}

__global__ void red_rows_scalar(float *C, uint32_t rows, int iters) {
    const int lane = threadIdx.x & 31, g = lane >> 3, j = lane & 7;
    const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    for (int it = 0; it < iters; ++it) {
        const uint32_t r = hash32(gw * 131071u + it * 4u + g) % rows;
        float *p = C + (size_t)r * 32 + j * 4;
#pragma unroll
        for (int q = 0; q < 4; ++q) atomicAdd(p + q, 1.f);
    }
}

// 64-byte rows (R = 16 floats): groups of 4 lanes, 8 rows per warp instruction
__global__ void gather_rows64(const float *__restrict__ B, uint32_t rows, int iters, float *sink) {
    const int lane = threadIdx.x & 31, g = lane >> 2, j = lane & 3;
    const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    float4 acc = make_float4(0, 0, 0, 0);
#pragma unroll 4
    for (int it = 0; it < iters; ++it) {
        const uint32_t r = hash32(gw * 131071u + it * 8u + g) % rows;
        float4 v = __ldg(reinterpret_cast<const float4 *>(B + (size_t)r * 16) + j);
        acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    if (acc.x + acc.y + acc.z + acc.w == 12345.f) *sink = acc.x;
}

__global__ void red_rows64(float *C, uint32_t rows, int iters) {
    const int lane = threadIdx.x & 31, g = lane >> 2, j = lane & 3;
    const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const float4 v = make_float4(1.f, 1.f, 1.f, 1.f);
    for (int it = 0; it < iters; ++it) {
        const uint32_t r = hash32(gw * 131071u + it * 8u + g) % rows;
        float *p = C + (size_t)r * 16 + j * 4;
        asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
    }
}

// gather 3 rows + red 2 rows per "entry": the c2 inner loop without index streaming
__global__ void mttkrp_like(const float *__restrict__ B, float *C, uint32_t rows, int iters) {
    const int lane = threadIdx.x & 31, g = lane >> 3, j = lane & 7;
    const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    for (int it = 0; it < iters; ++it) {
        const uint32_t h = gw * 131071u + it * 4u + g;
        const uint32_t r0 = hash32(h) % rows, r1 = hash32(h ^ 0x9e3779b9u) % rows, r2 = hash32(h ^ 0x85ebca6bu) % rows;
        float4 a = __ldg(reinterpret_cast<const float4 *>(B + (size_t)r0 * 32) + j);
        float4 b = __ldg(reinterpret_cast<const float4 *>(B + (size_t)r1 * 32) + j);
        float4 c = __ldg(reinterpret_cast<const float4 *>(B + (size_t)r2 * 32) + j);
        float4 u = make_float4(a.x * b.x, a.y * b.y, a.z * b.z, a.w * b.w);
        float4 w = make_float4(a.x * c.x, a.y * c.y, a.z * c.z, a.w * c.w);
        float *p1 = C + (size_t)r1 * 32 + j * 4, *p2 = C + (size_t)r2 * 32 + j * 4;
        asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p1), "f"(w.x), "f"(w.y), "f"(w.z), "f"(w.w) : "memory");
        asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p2), "f"(u.x), "f"(u.y), "f"(u.z), "f"(u.w) : "memory");
    }
}

// TMA-engine bulk reductions: each lane reduces one ROWB-byte row of smem into a random C row
template <int ROWB>
__global__ void bulk_red_rows(float *C, uint32_t rows, int iters) {
    __shared__ __align__(128) float buf[8][32][ROWB / 4];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = lane; i < 32 * ROWB / 4; i += 32) (&buf[warp][0][0])[i] = 1.f;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    const uint32_t src = (uint32_t)__cvta_generic_to_shared(&buf[warp][lane][0]);
    const uint32_t gt = blockIdx.x * blockDim.x + threadIdx.x;
    for (int it = 0; it < iters; ++it) {
        const uint32_t r = hash32(gt * 131071u + it) % rows;
        float *dst = C + (size_t)r * (ROWB / 4);
        asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(dst), "r"(src), "r"(ROWB) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 16;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// c2-shaped loop with the reductions issued by the TMA engine (bulk reduce from
// shared memory) instead of LSU REDs: does moving the scatter off the LSU path
// raise the combined gather+scatter rate?
__global__ void mttkrp_like_tma(const float *__restrict__ B, float *C, uint32_t rows, int iters) {
    __shared__ __align__(128) float stage[8][4][2][2][32];  // [warp][group][buffer][row][R]
    const int lane = threadIdx.x & 31, g = lane >> 3, j = lane & 7, w = threadIdx.x >> 5;
    const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    for (int it = 0; it < iters; ++it) {
        const int buf = it & 1;
        const uint32_t h = gw * 131071u + it * 4u + g;
        const uint32_t r0 = hash32(h) % rows, r1 = hash32(h ^ 0x9e3779b9u) % rows, r2 = hash32(h ^ 0x85ebca6bu) % rows;
        float4 a = __ldg(reinterpret_cast<const float4 *>(B + (size_t)r0 * 32) + j);
        float4 b = __ldg(reinterpret_cast<const float4 *>(B + (size_t)r1 * 32) + j);
        float4 c = __ldg(reinterpret_cast<const float4 *>(B + (size_t)r2 * 32) + j);
        float4 u = make_float4(a.x * b.x, a.y * b.y, a.z * b.z, a.w * b.w);
        float4 v = make_float4(a.x * c.x, a.y * c.y, a.z * c.z, a.w * c.w);
        if (lane % 8 == 0) asm volatile("cp.async.bulk.wait_group.read 2;" ::: "memory");  // buffer reuse
        __syncwarp();
        reinterpret_cast<float4 *>(stage[w][g][buf][0])[j] = v;
        reinterpret_cast<float4 *>(stage[w][g][buf][1])[j] = u;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (j == 0) {
            const uint32_t s0 = (uint32_t)__cvta_generic_to_shared(stage[w][g][buf][0]);
            const uint32_t s1 = (uint32_t)__cvta_generic_to_shared(stage[w][g][buf][1]);
            asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], 128;" ::"l"(C + (size_t)r1 * 32), "r"(s0) : "memory");
            asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], 128;" ::"l"(C + (size_t)r2 * 32), "r"(s1) : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
    }
    if (lane % 8 == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// shared-memory fp32 atomicAdd (a CAS loop on sm_100a) into a 64 KB private
// copy of C — the smem-privatisation alternative for small outputs (c5)
__global__ void smem_atomic_rows(float *out, int iters) {
    extern __shared__ float Cs[];  // 64 KB (dynamic): c5's C (1000 x 16)
    for (int i = threadIdx.x; i < 16384; i += blockDim.x) Cs[i] = 0.f;
    __syncthreads();
    const int lane = threadIdx.x & 31, j = lane & 3;
    const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    for (int it = 0; it < iters; ++it) {
        const uint32_t r = hash32(gw * 131071u + it * 8u + (lane >> 2)) % 1000;
#pragma unroll
        for (int q = 0; q < 4; ++q) atomicAdd(&Cs[r * 16 + j * 4 + q], 1.f);
    }
    __syncthreads();
    if (threadIdx.x == 0) out[blockIdx.x] = Cs[0];
}

int main() {
    int dev = 0, sms = 0, l2 = 0, smem = 0, clk = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    CK(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev));
    CK(cudaDeviceGetAttribute(&smem, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev));
    CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    float *sink;
    CK(cudaMalloc(&sink, 4));
    printf("{\"sms\": %d, \"l2_bytes\": %d, \"smem_per_sm\": %d, \"clock_khz\": %d", sms, l2, smem, clk);

    // 1) HBM stream read, 4 GiB
    {
        size_t bytes = size_t(4) << 30;
        float4 *a;
        CK(cudaMalloc(&a, bytes));
        CK(cudaMemset(a, 0, bytes));
        float best = 1e30f;
        for (int r = 0; r < 5; ++r) {
            CK(cudaEventRecord(e0));
            stream_read<<<sms * 8, 512>>>(a, bytes / 16, sink);
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            float ms;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            best = ms < best ? ms : best;
        }
        printf(", \"hbm_read_gbs\": %.1f", bytes / (best * 1e-3) / 1e9);
        CK(cudaFree(a));
    }
    // 2) L2 / HBM random 128-B row gathers for several table sizes
    const double tables_mb[] = {0.064, 0.64, 12.8, 64.0, 128.0, 512.0};
    printf(", \"gather_128B_rows_gbs\": {");
    for (int t = 0; t < 6; ++t) {
        uint32_t rows = (uint32_t)(tables_mb[t] * 1e6 / 128);
        float *B;
        CK(cudaMalloc(&B, (size_t)rows * 128));
        CK(cudaMemset(B, 0, (size_t)rows * 128));
        const int iters = 256, blocks = sms * 8, threads = 256;
        float best = 1e30f;
        for (int r = 0; r < 4; ++r) {
            CK(cudaEventRecord(e0));
            gather_rows<<<blocks, threads>>>(B, rows, iters, sink);
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            float ms;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            best = ms < best ? ms : best;
        }
        double bytes = (double)blocks * threads / 8 * iters * 128;
        printf("%s\"%.3fMB\": %.1f", t ? ", " : "", tables_mb[t], bytes / (best * 1e-3) / 1e9);
        CK(cudaFree(B));
    }
    printf("}");
    // 3) red.global.add.v4.f32 into random 128-B rows
    const double ctab_mb[] = {0.064, 0.64, 12.8, 128.0};
    printf(", \"red_v4_128B_rows_gbs\": {");
    for (int t = 0; t < 4; ++t) {
        uint32_t rows = (uint32_t)(ctab_mb[t] * 1e6 / 128);
        float *C;
        CK(cudaMalloc(&C, (size_t)rows * 128));
        CK(cudaMemset(C, 0, (size_t)rows * 128));
        const int iters = 128, blocks = sms * 8, threads = 256;
        float best = 1e30f;
        for (int r = 0; r < 4; ++r) {
            CK(cudaEventRecord(e0));
            red_rows<<<blocks, threads>>>(C, rows, iters);
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            float ms;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            best = ms < best ? ms : best;
        }
        double bytes = (double)blocks * threads / 8 * iters * 128;
        printf("%s\"%.3fMB\": %.1f", t ? ", " : "", ctab_mb[t], bytes / (best * 1e-3) / 1e9);
        CK(cudaFree(C));
    }
    printf("}");
    // 3a) the same for 64-byte rows (R = 16: c4, c5), gathers and red.v4
    const double t64_mb[] = {0.064, 0.64, 2.048, 12.8, 20.48};
    for (int kind = 0; kind < 2; ++kind) {
        printf(kind == 0 ? ", \"gather_64B_rows_gbs\": {" : ", \"red_v4_64B_rows_gbs\": {");
        for (int t = 0; t < 5; ++t) {
            uint32_t rows = (uint32_t)(t64_mb[t] * 1e6 / 64);
            float *X;
            CK(cudaMalloc(&X, (size_t)rows * 64));
            CK(cudaMemset(X, 0, (size_t)rows * 64));
            const int iters = kind == 0 ? 256 : 128, blocks = sms * 8, threads = 256;
            float best = 1e30f;
            for (int r = 0; r < 4; ++r) {
                CK(cudaEventRecord(e0));
                if (kind == 0) gather_rows64<<<blocks, threads>>>(X, rows, iters, sink);
                else red_rows64<<<blocks, threads>>>(X, rows, iters);
                CK(cudaEventRecord(e1));
                CK(cudaEventSynchronize(e1));
                float ms;
                CK(cudaEventElapsedTime(&ms, e0, e1));
                best = ms < best ? ms : best;
            }
            double bytes = (double)blocks * threads / 4 * iters * 64;
            printf("%s\"%.3fMB\": %.1f", t ? ", " : "", t64_mb[t], bytes / (best * 1e-3) / 1e9);
            CK(cudaFree(X));
        }
        printf("}");
    }
    // 3b) scalar atomicAdd, 12.8 MB
    {
        uint32_t rows = 100000;
        float *C;
        CK(cudaMalloc(&C, (size_t)rows * 128));
        CK(cudaMemset(C, 0, (size_t)rows * 128));
        const int iters = 64, blocks = sms * 8, threads = 256;
        float best = 1e30f;
        for (int r = 0; r < 3; ++r) {
            CK(cudaEventRecord(e0));
            red_rows_scalar<<<blocks, threads>>>(C, rows, iters);
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            float ms;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            best = ms < best ? ms : best;
        }
        double bytes = (double)blocks * threads / 8 * iters * 128;
        printf(", \"red_scalar_12.8MB_gbs\": %.1f", bytes / (best * 1e-3) / 1e9);
        CK(cudaFree(C));
    }
    // 4) same-row contention: all groups red into 1 row / 64 rows
    {
        float *C;
        CK(cudaMalloc(&C, 64 * 128));
        for (uint32_t rows : {1u, 64u}) {
            CK(cudaMemset(C, 0, 64 * 128));
            const int iters = 16, blocks = sms * 2, threads = 256;
            CK(cudaEventRecord(e0));
            red_rows<<<blocks, threads>>>(C, rows, iters);
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            float ms;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            double reds = (double)blocks * threads / 8 * iters;
            printf(", \"same_row_red_rows_per_us_%u\": %.1f", rows, reds / (ms * 1e3));
        }
        CK(cudaFree(C));
    }
    // 5) the c2-shaped inner loop without the index stream: 3 gathers + 2 reds per entry
    {
        uint32_t rows = 100000;
        float *B, *C;
        CK(cudaMalloc(&B, (size_t)rows * 128));
        CK(cudaMalloc(&C, (size_t)rows * 128));
        CK(cudaMemset(B, 0, (size_t)rows * 128));
        CK(cudaMemset(C, 0, (size_t)rows * 128));
        const int iters = 128, blocks = sms * 8, threads = 256;
        float best = 1e30f;
        for (int r = 0; r < 4; ++r) {
            CK(cudaEventRecord(e0));
            mttkrp_like<<<blocks, threads>>>(B, C, rows, iters);
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            float ms;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            best = ms < best ? ms : best;
        }
        double entries = (double)blocks * threads / 8 * iters;
        printf(", \"c2_like_entries_per_s\": %.4e, \"c2_like_ms_per_10M\": %.4f", entries / (best * 1e-3),
               best * 1e7 / entries);
        best = 1e30f;
        for (int r = 0; r < 4; ++r) {
            CK(cudaEventRecord(e0));
            mttkrp_like_tma<<<blocks, threads>>>(B, C, rows, iters);
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            float ms;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            best = ms < best ? ms : best;
        }
        printf(", \"c2_like_tma_red_ms_per_10M\": %.4f", best * 1e7 / entries);
        CK(cudaFree(B));
        CK(cudaFree(C));
    }
    // 6) bulk reductions (cp.reduce.async.bulk .add.f32) of 128-B / 64-B rows into 12.8 MB
    {
        uint32_t bytes_tab = 12800000;
        float *C;
        CK(cudaMalloc(&C, bytes_tab));
        CK(cudaMemset(C, 0, bytes_tab));
        const int iters = 64, blocks = sms * 4, threads = 256;
        float best = 1e30f;
        for (int r = 0; r < 3; ++r) {
            CK(cudaEventRecord(e0));
            bulk_red_rows<128><<<blocks, threads>>>(C, bytes_tab / 128, iters);
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            float ms;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            best = ms < best ? ms : best;
        }
        printf(", \"bulk_red_128B_rows_gbs\": %.1f", (double)blocks * threads * iters * 128 / (best * 1e-3) / 1e9);
        best = 1e30f;
        for (int r = 0; r < 3; ++r) {
            CK(cudaEventRecord(e0));
            bulk_red_rows<64><<<blocks, threads>>>(C, bytes_tab / 64, iters);
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            float ms;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            best = ms < best ? ms : best;
        }
        printf(", \"bulk_red_64B_rows_gbs\": %.1f", (double)blocks * threads * iters * 64 / (best * 1e-3) / 1e9);
        CK(cudaFree(C));
    }
    // 7) smem fp32 atomics (CAS loop) vs L2 red.v4: 64-B rows of a 64 KB C
    {
        float *o;
        CK(cudaMalloc(&o, sms * 4 * sizeof(float)));
        const int iters = 64, blocks = sms, threads = 1024;
        CK(cudaFuncSetAttribute(smem_atomic_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
        float best = 1e30f;
        for (int r = 0; r < 3; ++r) {
            CK(cudaEventRecord(e0));
            smem_atomic_rows<<<blocks, threads, 65536>>>(o, iters);
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            float ms;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            best = ms < best ? ms : best;
        }
        double bytes = (double)blocks * threads / 4 * iters * 64;   // 64-B row updates
        printf(", \"smem_cas_atomic_64B_rows_gbs\": %.1f", bytes / (best * 1e-3) / 1e9);
        CK(cudaFree(o));
    }
    printf("}\n");
    return 0;
}
