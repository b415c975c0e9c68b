// Do LSU reductions (red.global.add.v4.f32) and TMA-engine reductions
// (cp.reduce.async.bulk .add.f32) of random 128-byte rows share one limit, or
// can a kernel that issues both exceed what either reaches alone?
// One launch = 148*8 blocks of 256 threads; `tma_warps` of a block's 8 warps
// issue bulk reductions (one row per lane and iteration), the others red.v4
// (four rows per warp instruction).  Work per warp is sized so that both kinds
// reduce the same number of rows.  Prints one JSON line.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/microbench_red_mix tools/microbench_red_mix.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA error %s at %d\n", cudaGetErrorString(e_), __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
    return x;
}

__global__ void __launch_bounds__(256) red_mix(float *C, uint32_t rows, int rows_per_warp, int tma_warps) {
    __shared__ __align__(128) float buf[8][32][32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (warp < tma_warps) {
        for (int i = lane; i < 32 * 32; i += 32) (&buf[warp][0][0])[i] = 1.f;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        const uint32_t src = (uint32_t)__cvta_generic_to_shared(&buf[warp][lane][0]);
        for (int it = 0; it < rows_per_warp / 32; ++it) {
            const uint32_t r = hash32((gw * 32u + lane) * 131071u + it) % rows;
            float *dst = C + (size_t)r * 32;
            asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], 128;" ::"l"(dst), "r"(src) : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            asm volatile("cp.async.bulk.wait_group.read 16;" ::: "memory");
        }
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    } else {
        const int g = lane >> 3, j = lane & 7;
        const float4 v = make_float4(1.f, 1.f, 1.f, 1.f);
        for (int it = 0; it < rows_per_warp / 4; ++it) {
            const uint32_t r = hash32(gw * 131071u + it * 4u + g) % rows;
            float *p = C + (size_t)r * 32 + j * 4;
            asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
        }
    }
}

int main() {
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const uint32_t rows = 100000;  // 12.8 MB table (c2's C)
    float *C;
    CK(cudaMalloc(&C, (size_t)rows * 128));
    CK(cudaMemset(C, 0, (size_t)rows * 128));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    const int blocks = sms * 8, rows_per_warp = 4096;
    printf("{\"table_mb\": 12.8, \"blocks\": %d, \"rows_per_warp\": %d, \"gbs_by_tma_warps\": {", blocks, rows_per_warp);
    for (int tw = 0; tw <= 8; ++tw) {
        float best = 1e30f;
        for (int r = 0; r < 5; ++r) {
            CK(cudaEventRecord(e0));
            red_mix<<<blocks, 256>>>(C, rows, rows_per_warp, tw);
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            float ms;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            best = ms < best ? ms : best;
        }
        CK(cudaGetLastError());
        const double bytes = (double)blocks * 8 * rows_per_warp * 128;
        printf("%s\"%d\": %.1f", tw ? ", " : "", tw, bytes / (best * 1e-3) / 1e9);
    }
    printf("}}\n");
    return 0;
}
