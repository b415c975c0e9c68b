/*
 * Plain C use of the systec ABI (no Python, no torch): order-3 symmetric
 * MTTKRP of a tiny tensor through the host-buffer call, then the same through
 * a device plan.  Build (needs libsystec.so built in-tree and the CUDA runtime):
 *
 *   gcc -std=c11 -I include -I /usr/local/cuda/include examples/mttkrp_c.c -o /tmp/mttkrp_c \
 *       -L paper_2406_09266_b200 -lsystec -L /usr/local/cuda/lib64 -lcudart \
 *       -Wl,-rpath,$PWD/paper_2406_09266_b200
 *
 * The tensor is the hand-worked example of tests/golden/worked_example_n3.txt:
 * C = [[20, 6], [35, 7], [76, 12]].
 */
#include <stdio.h>

#include <cuda_runtime.h>

#include "systec.h"

#define CK(x)                                                                         \
    do {                                                                              \
        cudaError_t e_ = (x);                                                         \
        if (e_ != cudaSuccess) {                                                      \
            fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_));                  \
            return 1;                                                                 \
        }                                                                             \
    } while (0)

static int check(const char *what, const float *C, const float *want) {
    for (int k = 0; k < 6; ++k)
        if (C[k] != want[k]) {
            fprintf(stderr, "%s: C[%d] = %g, want %g\n", what, k, C[k], want[k]);
            return 1;
        }
    return 0;
}

int main(void) {
    const int32_t idx[4 * 3] = {0, 1, 2, 0, 0, 1, 1, 2, 2, 2, 2, 2};
    const float vals[4] = {1, 2, 3, 4};
    const float B[3 * 2] = {1, 1, 2, 1, 3, 1};
    float C[3 * 2] = {0};
    int rc = systec_mttkrp_host(3, 3, 4, idx, vals, B, 2, C, NULL);
    if (rc != SYSTEC_OK) {
        fprintf(stderr, "systec_mttkrp_host: %s\n", systec_status_string(rc));
        return 1;
    }
    const float want[6] = {20, 6, 35, 7, 76, 12};
    if (check("host call", C, want)) return 1;

    /* the same through a device plan: create (validate, canonicalise, sort,
     * statistics), execute on device buffers, copy C back */
    int32_t *d_idx;
    float *d_vals, *d_B, *d_C;
    CK(cudaMalloc((void **)&d_idx, sizeof(idx)));
    CK(cudaMalloc((void **)&d_vals, sizeof(vals)));
    CK(cudaMalloc((void **)&d_B, sizeof(B)));
    CK(cudaMalloc((void **)&d_C, sizeof(C)));
    CK(cudaMemcpy(d_idx, idx, sizeof(idx), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_vals, vals, sizeof(vals), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_B, B, sizeof(B), cudaMemcpyHostToDevice));
    systec_plan plan;
    rc = systec_plan_create(&plan, 3, 3, 4, d_idx, d_vals, NULL);
    if (rc == SYSTEC_OK) rc = systec_plan_execute(plan, d_B, 2, d_C, NULL);
    if (rc != SYSTEC_OK) {
        fprintf(stderr, "plan: %s\n", systec_status_string(rc));
        return 1;
    }
    float C2[3 * 2] = {0};
    CK(cudaMemcpy(C2, d_C, sizeof(C2), cudaMemcpyDeviceToHost));
    systec_plan_destroy(plan);
    cudaFree(d_idx);
    cudaFree(d_vals);
    cudaFree(d_B);
    cudaFree(d_C);
    if (check("device plan", C2, want)) return 1;
    printf("ok: C = [[%g, %g], [%g, %g], [%g, %g]] (host call and device plan)\n", C[0], C[1], C[2], C[3], C[4],
           C[5]);
    return 0;
}
