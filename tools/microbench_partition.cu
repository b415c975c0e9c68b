// Are row reductions faster when every row is owned by the issuing SM's own L2
// partition?  (half of a random row's reduction sectors cross
// the fabric between the two L2 partitions.)
//  1. calibration: one thread per SM times `atom.global.add.f32` (executed in
//     the owning partition, unlike a read, which the near partition caches)
//     on the first word of every 32-byte sector of a small table;
//  2. host: per SM, split its latencies at the largest gap around the median
//     into near / far; SMs are grouped by which sectors they see as near;
//  3. throughput: red.global.add.v4.f32 of whole 128-byte rows, each block
//     choosing rows near to its SM's partition / far from it / any.
// Prints one JSON line.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/microbench_partition tools/microbench_partition.cu
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA error %s at %d\n", cudaGetErrorString(e_), __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
    return x;
}
__device__ __forceinline__ uint32_t smid() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
    return r;
}

// one block per SM (the shared-memory request keeps two blocks off one SM)
__global__ void calibrate(float *T, int sectors, unsigned short *lat, int *sm_of_block) {
    extern __shared__ char pad[];
    if (threadIdx.x != 0) return;
    pad[0] = 0;
    const uint32_t sink = (uint32_t)__cvta_generic_to_shared(pad + 16);
    sm_of_block[blockIdx.x] = smid();
    for (int rep = 0; rep < 2; ++rep)  // second pass: the line is in L2 for sure
        for (int s = 0; s < sectors; ++s) {
            float *p = T + (size_t)s * 8;
            long long t0, t1;
            float old;
            asm volatile("mov.u64 %0, %%clock64;" : "=l"(t0)::"memory");
            asm volatile("atom.global.add.f32 %0, [%1], %2;" : "=f"(old) : "l"(p), "f"(0.0f) : "memory");
            // a store of the result issues only once it is back (in-order issue), the clock read after it
            asm volatile("st.volatile.shared.f32 [%0], %1;" ::"r"(sink), "f"(old) : "memory");
            asm volatile("mov.u64 %0, %%clock64;" : "=l"(t1)::"memory");
            if (rep) lat[(size_t)blockIdx.x * sectors + s] = (unsigned short)min(65535ll, t1 - t0);
        }
}

// mode 0: rows near to the block's SM, 1: far, 2: any
__global__ void __launch_bounds__(256) red_rows(float *T, const int *part_of_sm, const int *rows_of_part,
                                                const int *count_of_part, int rows_cap, int rows_all, int iters,
                                                int mode) {
    const int lane = threadIdx.x & 31, g = lane >> 3, j = lane & 7;
    const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int mine = part_of_sm[smid()];
    const int pick = mode == 0 ? mine : 1 - mine;
    const int *list = rows_of_part + (size_t)pick * rows_cap;
    const uint32_t n = mode == 2 ? rows_all : count_of_part[pick];
    const float4 v = make_float4(1.f, 1.f, 1.f, 1.f);
    for (int it = 0; it < iters; ++it) {
        const uint32_t k = hash32(gw * 131071u + it * 4u + g) % n;
        const uint32_t r = mode == 2 ? k : list[k];
        float *p = T + (size_t)r * 32 + j * 4;
        asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
    }
}

int main() {
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const int rows = 16384, sectors = rows * 4;  // 2 MB table
    float *T;
    CK(cudaMalloc(&T, (size_t)rows * 128));
    CK(cudaMemset(T, 0, (size_t)rows * 128));
    unsigned short *lat;
    int *smb;
    CK(cudaMalloc(&lat, (size_t)sms * sectors * 2));
    CK(cudaMalloc(&smb, sms * 4));
    CK(cudaFuncSetAttribute(calibrate, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    calibrate<<<sms, 32, 200 * 1024>>>(T, sectors, lat, smb);
    CK(cudaDeviceSynchronize());
    std::vector<unsigned short> h((size_t)sms * sectors);
    std::vector<int> hsm(sms);
    CK(cudaMemcpy(h.data(), lat, h.size() * 2, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(hsm.data(), smb, sms * 4, cudaMemcpyDeviceToHost));
    // per block (= SM): near/far split at the largest gap between the 25th and 75th percentile
    std::vector<std::vector<char>> near(sms, std::vector<char>(sectors));
    std::vector<int> thr(sms), lo_med(sms), hi_med(sms);
    for (int b = 0; b < sms; ++b) {
        std::vector<unsigned short> v(h.begin() + (size_t)b * sectors, h.begin() + (size_t)(b + 1) * sectors);
        std::sort(v.begin(), v.end());
        int best = 0, at = v[sectors / 2];
        for (int i = sectors / 4; i < 3 * sectors / 4; ++i)
            if (v[i + 1] - v[i] > best) { best = v[i + 1] - v[i]; at = (v[i + 1] + v[i]) / 2; }
        thr[b] = at;
        int nlo = 0;
        for (int s = 0; s < sectors; ++s) { near[b][s] = h[(size_t)b * sectors + s] <= at; nlo += near[b][s]; }
        lo_med[b] = v[std::max(0, nlo / 2)];
        hi_med[b] = v[std::min(sectors - 1, nlo + (sectors - nlo) / 2)];
    }
    // partition of an SM: agrees with block 0's view (0) or is its complement (1)
    std::vector<int> part_of_sm(256, 0);
    int agree_min = 100, part1 = 0;
    for (int b = 0; b < sms; ++b) {
        int same = 0;
        for (int s = 0; s < sectors; ++s) same += near[b][s] == near[0][s];
        const int pct = (int)(100.0 * same / sectors);
        const int p = pct >= 50 ? 0 : 1;
        part_of_sm[hsm[b]] = p;
        part1 += p;
        agree_min = std::min(agree_min, p ? 100 - pct : pct);
    }
    // rows whose four sectors share one owner, by block 0's view
    std::vector<int> rows_of_part(2 * rows);
    int cnt[2] = {0, 0}, split_rows = 0;
    for (int r = 0; r < rows; ++r) {
        const int s0 = near[0][4 * r] + near[0][4 * r + 1] + near[0][4 * r + 2] + near[0][4 * r + 3];
        if (s0 == 4) rows_of_part[cnt[0]++] = r;                 // near to partition 0
        else if (s0 == 0) rows_of_part[rows + cnt[1]++] = r;     // near to partition 1
        else ++split_rows;
    }
    printf("{\"sms\": %d, \"rows\": %d, \"block0_thr_cycles\": %d, \"block0_near_median\": %d, \"block0_far_median\": %d, "
           "\"sms_in_partition1\": %d, \"min_agreement_pct\": %d, \"rows_near_p0\": %d, \"rows_near_p1\": %d, \"rows_split\": %d",
           sms, rows, thr[0], lo_med[0], hi_med[0], part1, agree_min, cnt[0], cnt[1], split_rows);
    if (cnt[0] > 64 && cnt[1] > 64) {
        int *d_part, *d_rows, *d_cnt;
        CK(cudaMalloc(&d_part, 256 * 4));
        CK(cudaMalloc(&d_rows, 2 * rows * 4));
        CK(cudaMalloc(&d_cnt, 8));
        CK(cudaMemcpy(d_part, part_of_sm.data(), 256 * 4, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(d_rows, rows_of_part.data(), 2 * rows * 4, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(d_cnt, cnt, 8, cudaMemcpyHostToDevice));
        cudaEvent_t e0, e1;
        CK(cudaEventCreate(&e0));
        CK(cudaEventCreate(&e1));
        const int blocks = sms * 8, iters = 1024;
        const char *names[3] = {"near", "far", "any"};
        printf(", \"red_v4_128B_rows_gbs\": {");
        for (int mode = 0; mode < 3; ++mode) {
            float best = 1e30f;
            for (int r = 0; r < 5; ++r) {
                CK(cudaEventRecord(e0));
                red_rows<<<blocks, 256>>>(T, d_part, d_rows, d_cnt, rows, rows, iters, mode);
                CK(cudaEventRecord(e1));
                CK(cudaEventSynchronize(e1));
                float ms;
                CK(cudaEventElapsedTime(&ms, e0, e1));
                best = ms < best ? ms : best;
            }
            CK(cudaGetLastError());
            printf("%s\"%s\": %.1f", mode ? ", " : "", names[mode], (double)blocks * 32 * iters * 128 / (best * 1e-3) / 1e9);
        }
        printf("}");
    }
    printf("}\n");
    return 0;
}
