/*
 * uhstu_fp8.h — NEXT-2 of libuhstu: the layer's two projections in FP8
 * (arXiv 2602.16986 §4.2.2 "Mixed-Precision Training and Inference", P:151-166;
 * App. E.1).  "We execute both GEMMs in FP8, while preserving all
 * remaining operations in BF16"; the row-wise scaling and quantisation are
 * fused into the preceding layer-norm kernels (Fig. fp8); the post-attention
 * GEMM carries the 2-D residual bias in its epilogue.
 *
 * Format and scales (readings R17-R20): E4M3FN codes (1 byte, max 448),
 * round-to-nearest-even, saturating.  Activations: one fp32 scale per token row,
 * s = amax/448 (1 for an all-zero row), code = E4M3(v * (448/amax)) in fp32.
 * Weights: one scale per output column, stored transposed ([N][K], K-major).
 * D = diag(s_a) (q_a q_b^T) diag(s_b), fp32 accumulation (tcgen05 kind::f8f6f4).
 *
 * Conventions are those of uhstu.h (caller-owned memory, stream-ordered, all
 * checks before any launch, uh_status returns).  Codes are uint8 with row strides
 * in BYTES (multiples of 16); bf16 strides in elements (multiples of 8).
 */
#ifndef UHSTU_FP8_H
#define UHSTU_FP8_H
#include "uhstu.h"
#ifdef __cplusplus
extern "C" {
#endif

/* Eq. 1 + quantisation: x^ = LN(x) (fp32 in registers, never stored),
 * q[t,:] = E4M3 codes of x^[t,:], scale[t] = its row scale; mean / rstd [T] fp32
 * (may be NULL).  x bf16 [T,d] (ldx elements), q uint8 [T,d] (ldq bytes), d <= 2048,
 * d % 8 == 0.  Errors: UH_ERR_DIM (T < 0, d), UH_ERR_NULL, UH_ERR_ALIGNMENT. */
UH_API uh_status uh_ln_fwd_fp8(int64_t T, int d, const void* x, int64_t ldx, const float* w, const float* b,
                               float eps, uint8_t* q, int64_t ldq, float* scale, float* mean, float* rstd,
                               void* stream);

/* Eq. 4 inner + quantisation: Y = LN(A) (.) U quantised per row as
 * above.  A, U bf16 [T,d] (lda, ldu elements; U may be the U block of UVQK). */
UH_API uh_status uh_gated_norm_fwd_fp8(int64_t T, int d, const void* A, int64_t lda, const void* U, int64_t ldu,
                                       const float* w, const float* b, float eps, uint8_t* q, int64_t ldq,
                                       float* scale, float* mean, float* rstd, void* stream);

/* Weight quantisation (R18): W bf16 [K,N] (ldw elements) -> qt uint8 [N,K] (W^T,
 * K-major, ldq bytes) and scale[N] (one per output column).  Run once per weight
 * update.  Errors: UH_ERR_DIM, UH_ERR_NULL, UH_ERR_ALIGNMENT. */
UH_API uh_status uh_quant_weight_fp8(int K, int N, const void* W, int64_t ldw, uint8_t* qt, int64_t ldq,
                                     float* scale, void* stream);

/* FP8 projection: acc = q_a[M,K] q_b[N,K]^T (fp32),
 * h = acc * sa[m] * sb[n] + bias[n] (bias may be NULL);
 * epi 0: out = h (+ resid[m,n] when resid != NULL: the 2-D bias of f2, Eq. 5), bf16;
 * epi 1: out = silu(h) (f1 + phi1, Eq. 2), bf16.
 * K % 128 == 0, N % 128 == 0, M >= 0.  out / resid bf16 [M,N] (ld elements).
 * Errors: UH_ERR_DIM, UH_ERR_NULL, UH_ERR_ALIGNMENT, UH_ERR_UNSUPPORTED (K, N). */
UH_API uh_status uh_gemm_fp8(int M, int N, int K, const uint8_t* qa, int64_t lda, const float* sa,
                             const uint8_t* qb, int64_t ldb, const float* sb, int epi, void* out, int64_t ldo,
                             const float* bias, const void* resid, int64_t ldr, void* stream);

/* Quantised weights of one layer (uh_quant_weight_fp8 of p->w1 [d,4d] and p->w2 [d,d]). */
typedef struct {
    const uint8_t* w1t;  const float* s1;   /* [4d][d] codes, [4d] scales */
    const uint8_t* w2t;  const float* s2;   /* [d][d] codes,  [d] scales  */
} uh_fp8_weights;

/* The layer forward of uh_layer_fwd (Eqs. 1-5) with both projections in FP8
 * (P:156): LN+quant -> FP8 f1 + SiLU -> attention (bf16, unchanged) -> gated
 * norm+quant -> FP8 f2 + b2 + x.  dtype is UH_BF16; the workspace is the one
 * uh_layer_workspace_bytes(..., UH_BF16, 0, ...) reports; saved as in uh_layer_fwd
 * (attn and the LayerNorm statistics; the bf16 backward can consume them). */
UH_API uh_status uh_layer_fwd_fp8(const uh_jagged* jag, uh_mask m, const uh_layer_params* p,
                                  const uh_fp8_weights* qw, const void* x, void* out, uh_layer_saved* saved,
                                  void* ws, size_t ws_bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif
