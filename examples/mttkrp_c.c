/*
 * Plain C use of the systec ABI (no Python, no torch): order-3 symmetric
 * MTTKRP of a tiny tensor through the host-buffer call, then the same through
 * a device plan.  Build (needs libsystec.so built in-tree and the CUDA runtime):
 *
 *   gcc -std=c11 -I include examples/mttkrp_c.c -o /tmp/mttkrp_c \
 *       -L paper_2406_09266_b200 -lsystec -L /usr/local/cuda/lib64 -lcudart \
 *       -Wl,-rpath,$PWD/paper_2406_09266_b200
 *
 * The tensor is the hand-worked example of tests/golden/worked_example_n3.txt:
 * C = [[20, 6], [35, 7], [76, 12]].
 */
#include <stdio.h>

#include "systec.h"

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
    for (int k = 0; k < 6; ++k)
        if (C[k] != want[k]) {
            fprintf(stderr, "C[%d] = %g, want %g\n", k, C[k], want[k]);
            return 1;
        }
    printf("ok: C = [[%g, %g], [%g, %g], [%g, %g]]\n", C[0], C[1], C[2], C[3], C[4], C[5]);
    return 0;
}
