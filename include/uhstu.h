/*
 * uhstu.h — C ABI of libuhstu, the B200 (sm_100a) hot path of ULTRA-HSTU
 * (arXiv 2602.16986): the jagged, semi-local HSTU attention layer, forward and
 * backward, plus the host partitioner that shards a jagged batch across GPUs.
 *
 * Citations: "P:n" = line n of PAPER.md (the paper's LaTeX source), "R<k>" =
 * reading k in DESIGN.md §3 (where the paper is silent, garbled or ambiguous).
 *
 * Conventions (all entry points):
 *  - Every function is extern "C", never throws and returns uh_status.
 *  - The caller owns ALL memory, including the workspace.  The library never
 *    allocates device memory, never frees, and retains no pointer after it
 *    returns; work is enqueued on `stream` (a cudaStream_t passed as void*,
 *    NULL = legacy default stream) and buffers must stay alive until the stream
 *    has passed it.
 *  - Activations are row-major [T, width] with an explicit row stride `ld`
 *    (elements).  T = total tokens of the jagged batch; rows of sequence i are
 *    [offsets[i], offsets[i+1]) in time-ascending order (index 0 = earliest).
 *  - dtype UH_BF16: activations/weights bf16, fp32 accumulation (tcgen05 path).
 *    dtype UH_F32: the fp32 SIMT verification build (same ABI, fp32 everywhere).
 *    LayerNorm parameters, rab tables and parameter gradients are always fp32.
 *  - Alignment: device pointers 16-byte aligned; bf16 row strides multiples of
 *    8 elements, fp32 strides multiples of 4 (TMA / 16-byte vector access).
 *    Violations return UH_ERR_ALIGNMENT before anything is launched.
 *  - All argument checks run before any launch: a failing call has no side
 *    effects.  Launch failures return UH_ERR_CUDA with the CUDA error string in
 *    uh_last_error(); asynchronous device faults surface at the caller's next
 *    synchronisation.
 *  - Thread-safe and stateless apart from idempotent per-device lazy init
 *    (kernel attributes, driver entry points).
 *  - B = 0 and L_i = 0 are valid no-ops.
 */
#ifndef UHSTU_H
#define UHSTU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define UH_API __attribute__((visibility("default")))
#else
#define UH_API
#endif

#define UH_ABI_VERSION 1
#define UH_WINDOW_FULL 2147483647 /* mask.window value meaning "no window limit" (full causal) */

typedef enum {
    UH_OK = 0,
    UH_ERR_DIM = 1,            /* sizes inconsistent (offsets length, total_tokens, ...)      */
    UH_ERR_DOMAIN = 2,         /* value out of domain (negative length, window, heads ...)     */
    UH_ERR_SHAPE = 3,          /* head_dim * num_heads != d, unsupported head_dim              */
    UH_ERR_CACHE_MISMATCH = 4, /* saved set missing / mismatched between forward and backward  */
    UH_ERR_ALIGNMENT = 5,      /* pointer or stride misaligned                                 */
    UH_ERR_WORKSPACE = 6,      /* workspace NULL or smaller than the *_workspace_bytes query   */
    UH_ERR_UNSUPPORTED = 7,    /* valid request this build does not implement                  */
    UH_ERR_CUDA = 8,           /* a CUDA call failed; see uh_last_error()                      */
    UH_ERR_NULL = 9            /* required pointer is NULL                                     */
} uh_status;

typedef enum { UH_BF16 = 0, UH_F32 = 1 } uh_dtype;

UH_API const char* uh_status_string(uh_status s);
/* Detail of the last failure on the calling thread (empty string if none). */
UH_API const char* uh_last_error(void);
UH_API int uh_abi_version(void);

/* ---------------------------------------------------------------------------
 * Jagged batch ("X_i in R^{L_i x d}"; "fully jagged tensor").
 * offsets[0] = 0, non-decreasing, offsets[num_seqs] = total_tokens.
 * `offsets` is the device copy used by kernels; `host_offsets` the identical
 * host copy read by the host tile scheduler (F0) and by validation.
 * max_len must equal max_i (offsets[i+1]-offsets[i]).
 * ------------------------------------------------------------------------- */
typedef struct {
    int32_t num_seqs;
    int32_t max_len;
    int64_t total_tokens;
    const int32_t* offsets;      /* device, [num_seqs+1] */
    const int32_t* host_offsets; /* host,   [num_seqs+1] */
} uh_jagged;

/* ---------------------------------------------------------------------------
 * Semi-local mask (§4.2.1), time-ascending reading R1-R4:
 *   key k is visible to query q (same sequence) iff
 *       k <= q  and  ( q - k <= window  or  k < n_global ).
 * window = UH_WINDOW_FULL gives the full causal mask of Eq. 3.
 * window >= 0, n_global >= 0, else UH_ERR_DOMAIN.
 * ------------------------------------------------------------------------- */
typedef struct {
    int32_t window;   /* K1 (inclusive: the query sees itself and K1 predecessors, R2) */
    int32_t n_global; /* K2 (keys 0..K2-1 of each sequence are global, R3)             */
} uh_mask;

/* ---------------------------------------------------------------------------
 * Attention descriptor.  Per head h (columns [h*head_dim, (h+1)*head_dim)):
 *   s(q,k) = alpha * <Q_q, K_k> + pos_bias[min(q-k, pos_bias_len-1)]
 *                              + time_bias[min(time_bias_len-1, floor(log2(max(t_q-t_k,1))))]
 *   A_q    = sum_{k visible} silu(s(q,k)) / norm_n * V_k                (Eq. 3)
 * The bias terms are the north star's relative position/time bias (R7; not in
 * the paper) and are shared by all heads; NULL tables switch them off.
 * norm_n is the 1/N normaliser (R5), alpha the score scale (R6).
 * head_dim in {32, 64, 128} (bf16 tcgen05 kernels require 128; 32/64 run the
 * fp32 verification build only).  time_bias_len <= 32 (buckets of log2 seconds).
 * pos_bias_len is any P >= 1 (offsets q - k >= P - 1 share the last entry); the bf16
 * path reads it through an extended copy built in the workspace each call.
 * ------------------------------------------------------------------------- */
typedef struct {
    int32_t num_heads;
    int32_t head_dim;
    float alpha;
    float norm_n;                /* > 0 */
    const float* pos_bias;       /* device fp32 [pos_bias_len] or NULL  */
    int32_t pos_bias_len;
    const float* time_bias;      /* device fp32 [time_bias_len] or NULL */
    int32_t time_bias_len;
    const int64_t* timestamps;   /* device int64 [total_tokens]; required iff time_bias; non-decreasing per sequence */
} uh_attn_desc;

/* Number of visible (q,k) pairs of a length-L sequence (closed form; host). */
UH_API int64_t uh_mask_nnz(uh_mask m, int64_t L);
/* Sum over the batch of uh_mask_nnz (host; reads host_offsets). */
UH_API int64_t uh_batch_nnz(const uh_jagged* jag, uh_mask m);

/* Workspace bytes for uh_attn_fwd (backward=0) or uh_attn_bwd (backward=1).  The bf16
 * backward's workspace holds the tile schedule and an fp32 [T, H*head_dim] dQ accumulator
 * (4 bytes per token and dQ column; zeroed inside the call), so it is ~T*H*head_dim*4 bytes. */
UH_API uh_status uh_attn_workspace_bytes(const uh_jagged* jag, uh_mask m, const uh_attn_desc* desc,
                                  uh_dtype dtype, int backward, size_t* bytes);

/* Attention forward (Eq. 3 with the SLA mask).  q, k, v: [T, >= H*dh] with row
 * stride ld_qkv (they may be column blocks of one fused [T,4d] buffer);
 * out: [T, >= H*dh], row stride ld_out, overwritten on every real row. */
UH_API uh_status uh_attn_fwd(const uh_jagged* jag, uh_mask m, const uh_attn_desc* desc, uh_dtype dtype,
                      const void* q, const void* k, const void* v, int64_t ld_qkv,
                      void* out, int64_t ld_out, void* ws, size_t ws_bytes, void* stream);

/* Attention backward (Listing 1 "attention_backward(dattn, q, k, v)").
 * dout: dL/dA, row stride ld_dout.  dq, dk, dv: overwritten, row stride ld_grad.
 * bf16: one key-major kernel computes dK, dV and the dQ partials (reduced into the
 * workspace's fp32 accumulator), then a finish kernel writes dq; the call is stream-ordered
 * and CUDA-graph capturable (a cudaMemsetAsync zeroes the accumulator).
 * dpos_bias / dtime_bias: fp32, ACCUMULATED into (caller zeroes); may be NULL
 * when the matching table is NULL. */
UH_API uh_status uh_attn_bwd(const uh_jagged* jag, uh_mask m, const uh_attn_desc* desc, uh_dtype dtype,
                      const void* q, const void* k, const void* v, int64_t ld_qkv,
                      const void* dout, int64_t ld_dout,
                      void* dq, void* dk, void* dv, int64_t ld_grad,
                      float* dpos_bias, float* dtime_bias,
                      void* ws, size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------------
 * The HSTU layer, Eqs. 1-5 in Listing 1's order:
 *   x^  = LN(x; ln1_w, ln1_b)                         (Eq. 1, LayerNorm R9)
 *   UVQK = silu(x^ W1 + b1)    W1 [d,4d] cols U|V|Q|K (Eq. 2, R11)
 *   A   = attention(Q, K, V)                          (Eq. 3)
 *   Y   = LN(A; ln2_w, ln2_b) (.) U                   (Eq. 4, gated norm)
 *   out = Y W2 + b2 + x         W2 [d,d]              (Eqs. 4-5, 2-D residual bias)
 * w1, w2: device, dtype as requested, row-major.  b1, b2 nullable (zero).
 * ------------------------------------------------------------------------- */
typedef struct {
    const float* ln1_w; const float* ln1_b;
    const void* w1;     const float* b1;
    const float* ln2_w; const float* ln2_b;
    const void* w2;     const float* b2;
    uh_attn_desc attn;
    float eps;          /* LayerNorm epsilon (1e-6) */
} uh_layer_params;

/* Saved-activation set for the rematerialising backward (Listing 1
 * saves {x, u, attn}; this build saves {x (the caller's input), attn} plus the
 * LayerNorm statistics and rematerialises U with V,Q,K — DESIGN.md §5).
 * attn: [T,d] (dtype), ld = d.  Stats fp32 [T].  All caller-owned.
 * fingerprint: written by uh_layer_fwd / uh_layer_fwd_fp8 (a hash of the host offsets,
 * the mask, the attention descriptor's shape and scalars, eps and dtype); uh_layer_bwd
 * returns UH_ERR_CACHE_MISMATCH when it differs from the backward call's (S:303
 * "wrong cache variant"), e.g. a backward with another mask than its forward. */
typedef struct {
    void* attn;
    float* ln1_mean; float* ln1_rstd;
    float* ln2_mean; float* ln2_rstd;
    uint64_t fingerprint;
} uh_layer_saved;

/* Parameter gradients, fp32, same shapes as the parameters.  b1/b2/pos/time may
 * be NULL when the parameter is absent.  Sums over all tokens of the batch. */
typedef struct {
    float* ln1_w; float* ln1_b;
    float* w1;    float* b1;
    float* ln2_w; float* ln2_b;
    float* w2;    float* b2;
    float* pos_bias; float* time_bias;
} uh_layer_grads;

UH_API uh_status uh_layer_workspace_bytes(const uh_jagged* jag, uh_mask m, const uh_layer_params* p,
                                   uh_dtype dtype, int backward, size_t* bytes);

/* x, out: [T,d] row stride d.  saved = NULL => inference (nothing saved). */
UH_API uh_status uh_layer_fwd(const uh_jagged* jag, uh_mask m, const uh_layer_params* p, uh_dtype dtype,
                       const void* x, void* out, uh_layer_saved* saved,
                       void* ws, size_t ws_bytes, void* stream);

/* dout: dL/dout [T,d]; dx: [T,d] overwritten (includes the residual "dx += dout",
 * P:577).  accumulate=0 overwrites *grads, 1 adds into them. */
UH_API uh_status uh_layer_bwd(const uh_jagged* jag, uh_mask m, const uh_layer_params* p, uh_dtype dtype,
                       const void* x, const uh_layer_saved* saved, const void* dout, void* dx,
                       uh_layer_grads* grads, int accumulate,
                       void* ws, size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------------
 * Jagged gather / scatter (P:190 jagged tensors).
 * Row bytes (width * elem_bytes) must be a multiple of 8 and x / y 16-byte
 * aligned (UH_ERR_ALIGNMENT); 16-byte multiples take the vectorised path, 8-byte
 * rows (e.g. int64 timestamps, width 1) one lane per row.
 * ------------------------------------------------------------------------- */
/* Pack the rows of sequences seq_ids_host[0..n) of `src` (row width `width`
 * elements of `elem_bytes` bytes, row stride ld_x) contiguously into y (row
 * stride width).  dst_offsets_host receives the packed offsets [n+1] (host),
 * dst_offsets_dev (device, may be NULL) a device copy. */
UH_API uh_status uh_jagged_gather(const uh_jagged* src, const int32_t* seq_ids_host, int32_t n,
                           const void* x, int64_t ld_x, int64_t width, int32_t elem_bytes,
                           void* y, int32_t* dst_offsets_host, int32_t* dst_offsets_dev,
                           void* stream);
/* Keep the latest min(L_i, l_keep) rows of each sequence (attention truncation,
 * P:198-199 "truncating latest UIH of length L'").  dst_offsets_* as above. */
UH_API uh_status uh_jagged_slice_latest(const uh_jagged* src, int32_t l_keep,
                                 const void* x, int64_t ld_x, int64_t width, int32_t elem_bytes,
                                 void* y, int32_t* dst_offsets_host, int32_t* dst_offsets_dev,
                                 void* stream);
/* jagged [T,width] <-> padded [B, max_len, width] (padding rows filled with zero
 * bytes set to 0 on jagged->padded). */
UH_API uh_status uh_jagged_to_padded(const uh_jagged* src, const void* x, int64_t width, int32_t elem_bytes,
                              int32_t max_len, void* y, void* stream);
UH_API uh_status uh_padded_to_jagged(const uh_jagged* dst, const void* y, int64_t width, int32_t elem_bytes,
                              int32_t max_len, void* x, void* stream);

/* ---------------------------------------------------------------------------
 * Token-balanced partitioner (host, deterministic).
 * cost(L) = 4*(2 L d 4d) + 3*(2 L d d) + 14 * head_dim * H * uh_mask_nnz(m, L)
 * (the layer step's flops on the sequence: f1, remat f1, dW1, dx^; f2, dY, dW2; attention);
 * LPT: sequences by (cost desc, id asc), each to the least-loaded rank (lowest
 * id on ties).  Outputs rank_of_seq[B] and rank_cost[world] (host).
 * The load notion follows LBSL's "sum n_u^gamma".
 * ------------------------------------------------------------------------- */
UH_API uh_status uh_partition_lpt(const int32_t* lengths, int32_t B, int32_t world, uh_mask m,
                           int32_t d, int32_t num_heads, int32_t* rank_of_seq, double* rank_cost);

#ifdef __cplusplus
}
#endif
#endif /* UHSTU_H */
