/*
 * uhstu_testing.h — test hooks of libuhstu (not part of the product ABI).
 * Exposes the internal projection GEMM so its tcgen05 descriptor / major /
 * epilogue variants can be checked element by element against a reference.
 */
#ifndef UHSTU_TESTING_H
#define UHSTU_TESTING_H
#include "uhstu.h"
#ifdef __cplusplus
extern "C" {
#endif
/* C[M,N] = A * B with A stored [M][K] (a_mn=0) or [K][M] (a_mn=1), B stored [N][K]
 * (b_mn=0) or [K][N] (b_mn=1).  epi: 0 = out0 = C + bias + resid (dtype),
 * 1 = out0 = silu(C + bias), out1 = silu'(C + bias) (dtype), 2 = out0 += C (fp32).
 * cta_pair: 0 = single-CTA tiles (the layer's path), 1 = cta_group::2 pair tiles for
 * MN-major B, 2 = pair tiles for both B majors (where the shape is eligible). */
UH_API uh_status uh_test_gemm(int M, int N, int K, const void* A, int64_t lda, int a_mn, const void* B, int64_t ldb,
                              int b_mn, int epi, void* out0, int64_t ld0, void* out1, int64_t ld1, const float* bias,
                              const void* resid, int64_t ldr, uh_dtype dtype, int cta_pair, void* stream);
/* Number of kernels the library has launched in this process (all entry points). */
UH_API long long uh_test_launch_count(void);
#ifdef __cplusplus
}
#endif
#endif
