// internal.h — host-side internal interface between the C-ABI layer (abi.cu) and
// the kernel launchers.  Not exported; not part of include/uhstu.h.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/uhstu.h"

namespace uh {

// ------------------------------------------------------------------ errors
void set_error(const std::string& msg);
uh_status fail(uh_status s, const std::string& msg);
uh_status cuda_fail(cudaError_t e, const char* where);
#define UH_CUDA(call)                                             \
    do {                                                          \
        cudaError_t e_ = (call);                                  \
        if (e_ != cudaSuccess) return ::uh::cuda_fail(e_, #call); \
    } while (0)
#define UH_TRY(call)                      \
    do {                                  \
        uh_status s_ = (call);            \
        if (s_ != UH_OK) return s_;       \
    } while (0)

// bf16 2-D tensor map, 128-byte swizzle, box {box_inner, box_outer}
uh_status make_tmap_bf16(CUtensorMap* map, const void* ptr, uint64_t inner, uint64_t outer, uint64_t ld_elems,
                         uint32_t box_inner, uint32_t box_outer, int swizzle_bytes = 128);
// 8-bit (E4M3) 2-D tensor map, 128-byte swizzle; ld in bytes
uh_status make_tmap_u8(CUtensorMap* map, const void* ptr, uint64_t inner, uint64_t outer, uint64_t ld_bytes,
                       uint32_t box_inner, uint32_t box_outer);
// fp32 2-D tensor map, no swizzle (TMA reduce-add targets)
uh_status make_tmap_f32(CUtensorMap* map, const void* ptr, uint64_t inner, uint64_t outer, uint64_t ld_elems,
                        uint32_t box_inner, uint32_t box_outer);
int num_sms();
// the ABI's jagged-descriptor validation (abi.cu), shared by the other exported entry points
uh_status validate_jagged(const uh_jagged* j, bool need_device);
// every kernel launch of the library is counted (bench.py reports gpu_launches from it)
void note_launch();

// ------------------------------------------------------------------ GEMM
// C[M,N] = A[M,K] * B[K,N].  a_mn: A stored [K][M] (else [M][K]); b_mn: B stored
// [K][N] (else [N][K]).  Epilogue per gemm_sm100.cuh (EPI_BF16 / EPI_SILU / EPI_F32).
constexpr int kGemmPairDefault = 0;   // compile-time choice of the product path (no runtime dispatch)
struct GemmDesc {
    int M = 0, N = 0, K = 0;
    const void* A = nullptr; int64_t lda = 0; bool a_mn = false;
    const void* B = nullptr; int64_t ldb = 0; bool b_mn = false;
    int epi = 0;
    void* out0 = nullptr; int64_t ld0 = 0;
    void* out1 = nullptr; int64_t ld1 = 0;
    const float* bias = nullptr;
    const void* resid = nullptr; int64_t ldr = 0;
    float* colsum = nullptr;   // EPI_F32 only: += column sums of B (fused bias gradient)
    int pair = kGemmPairDefault;   // cta_group::2 pair tiles: 0 off, 1 MN-major B only, 2 both majors
};
uh_status gemm_run(const GemmDesc& g, uh_dtype dt, cudaStream_t st);
// NEXT-2: D = diag(sa) (A B) diag(sb) (+ bias)(+ resid) with A [M,K] and B^T [N,K] E4M3, K-major,
// epi EPI_BF16 or EPI_SILU (g.A / g.B the codes, lda / ldb in bytes); K % 128 == 0, N % 128 == 0
uh_status gemm_fp8_run(const GemmDesc& g, const float* sa, const float* sb, cudaStream_t st);

// ------------------------------------------------------------------ norms (norm.cu)
// x^ = LN(x) with stats out (mean/rstd may be null)
uh_status ln_fwd(uh_dtype dt, int64_t T, int d, const void* x, int64_t ldx, const float* w, const float* b, float eps,
                 void* y, int64_t ldy, float* mean, float* rstd, cudaStream_t st);
// x^ = (x - mean) * rstd * w + b from saved statistics (remat)
uh_status ln_apply(uh_dtype dt, int64_t T, int d, const void* x, int64_t ldx, const float* w, const float* b,
                   const float* mean, const float* rstd, void* y, int64_t ldy, cudaStream_t st);
// Y = LN(A) (.) U, stats out
uh_status gated_norm_fwd(uh_dtype dt, int64_t T, int d, const void* A, int64_t lda, const void* U, int64_t ldu,
                         const float* w, const float* b, float eps, void* Y, int64_t ldy, float* mean, float* rstd,
                         cudaStream_t st);
// NEXT-2: LN / gated norm with the row-wise E4M3 quantisation fused (bf16 in, codes [T,d] + scale [T])
uh_status ln_fwd_fp8(int64_t T, int d, const void* x, int64_t ldx, const float* w, const float* b, float eps,
                     uint8_t* q, int64_t ldq, float* scale, float* mean, float* rstd, cudaStream_t st);
uh_status gated_norm_fwd_fp8(int64_t T, int d, const void* A, int64_t lda, const void* U, int64_t ldu,
                             const float* w, const float* b, float eps, uint8_t* q, int64_t ldq, float* scale,
                             float* mean, float* rstd, cudaStream_t st);
// W [K,N] bf16 -> W^T codes [N,K] + per-column scales [N]
uh_status quant_weight_fp8(int K, int N, const void* W, int64_t ldw, uint8_t* qt, int64_t ldq, float* scale,
                           cudaStream_t st);
// gated norm backward: dA, dH_U = (dY (.) A^) (.) G_U, Y (recomputed), dw, db (+=)
uh_status gated_norm_bwd(uh_dtype dt, int64_t T, int d, const void* dY, int64_t lddy, const void* A, int64_t lda,
                         const void* U, int64_t ldu, const void* GU, int64_t ldg, const float* w, const float* b,
                         const float* mean, const float* rstd, void* dA, int64_t ldda, void* dHU, int64_t ldh,
                         void* Y, int64_t ldy, float* dw, float* db, cudaStream_t st);
// dx = LN_bwd(dxh) + dres ; dw, db (+=)
uh_status ln_bwd(uh_dtype dt, int64_t T, int d, const void* dxh, int64_t ldg, const void* x, int64_t ldx,
                 const float* w, const float* mean, const float* rstd, const void* dres, int64_t ldr, void* dx,
                 int64_t lddx, float* dw, float* db, cudaStream_t st);
// out[c] (+)= sum_rows M[r, c]
uh_status colsum(uh_dtype dt, int64_t T, int n, const void* M, int64_t ldm, float* out, cudaStream_t st);
// dst = bf16/f32(acc * G) elementwise over [T, n]

// ------------------------------------------------------------------ attention
struct AttnCall {
    const uh_jagged* jag;
    uh_mask mask;
    const uh_attn_desc* desc;
    const void *q, *k, *v; int64_t ld_qkv;
    // forward
    void* out; int64_t ld_out;
    // backward
    const void* dout; int64_t ld_dout;
    void *dq, *dk, *dv; int64_t ld_grad;
    const void *gq, *gk, *gv; int64_t ld_gate;  // optional silu'(h) gates multiplied into dq/dk/dv (layer path)
    float *dpos, *dts;
    void* ws; size_t ws_bytes;
    cudaStream_t st;
};
size_t attn_ws_bytes(const uh_jagged* jag, uh_mask m, const uh_attn_desc* desc, uh_dtype dt, int backward);
uh_status attn_fwd_run(const AttnCall& c, uh_dtype dt);
uh_status attn_bwd_run(const AttnCall& c, uh_dtype dt);

}  // namespace uh
