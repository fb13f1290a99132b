/*
 * uhstu_mot.h — NEXT-4: the Mixture of Transducers fusion of libuhstu (arXiv 2602.16986
 * §4.3, "MoT processes multiple distinct input sequences through separate
 * transducers and subsequently fuses the learned user embeddings"; App. A P:390-392 "two
 * specialized HSTU modules: one for engagement events and one for consumption events").
 * Readings R28-R30 of DESIGN.md; conventions of uhstu.h (caller-owned memory, stream
 * ordering, every check before any launch, failing calls have no side effects).
 *
 * A MoT model runs K branches.  Branch k is a stack of uh_layer_fwd / uh_layer_bwd calls on
 * its own jagged batch (its own parameters, depth and mask, R30); every branch holds the same
 * B users in the same order.  The last n_cand rows of every sequence are the candidate
 * positions (R29: P:74 candidates x_j, P:104 candidates inside the sequence).  The fusion
 * (R28) maps the branches' final states X_k [T_k, d] to one embedding per candidate:
 *
 *     Z = [ X_0[cand] | X_1[cand] | ... | X_{K-1}[cand] ]   [C, K d], C = B n_cand
 *     E = Z W_f + b_f                                          [C, d]
 *
 * with X_k[cand] row (b n_cand + j) = X_k row offsets_k[b+1] - n_cand + j.  The backward of
 * the loss sum(dE (.) E) gives the fusion's parameter gradients and each branch's output
 * gradient, the seed of that branch's uh_layer_bwd chain:
 *
 *     dW_f = Z^T dE,  db_f = sum_rows dE,
 *     dX_k = 0 except dX_k[cand] = (dE W_f^T)[:, k d : (k+1) d].
 *
 * Kernels: a candidate gather / scatter (one warp per row, 16-byte vectors, HBM bound) and the
 * tcgen05 GEMMs of the layer (E: bias epilogue; dW_f: split-K fp32 with the bias column sum
 * fused when d and K d are multiples of 256, else a separate column-sum pass).
 */
#ifndef UHSTU_MOT_H
#define UHSTU_MOT_H

#include "uhstu.h"

#ifdef __cplusplus
extern "C" {
#endif

/* One branch's final states: x [T_k, d] (dtype of the call) with row stride ld (elements),
 * over the jagged batch jag (device + host offsets as in uhstu.h). */
typedef struct {
    const uh_jagged* jag;
    const void* x;
    int64_t ld;
} uh_mot_branch;

/* Workspace of uh_mot_fuse_fwd (backward = 0: Z, C K d elements) or uh_mot_fuse_bwd
 * (backward = 1: Z and dZ, 2 C K d elements), dtype-sized, rounded to 256 bytes. */
UH_API uh_status uh_mot_workspace_bytes(int32_t n_branches, const uh_mot_branch* branches, int32_t n_cand,
                                        int32_t d, uh_dtype dtype, int backward, size_t* bytes);

/* E [C, d] (row stride d, dtype) = concat_k X_k[cand] W_f + b_f.
 * w_f: device [n_branches d, d] row-major (dtype); b_f: device fp32 [d] or NULL (zero).
 * Errors (before any launch): UH_ERR_NULL (branches, a jag / x, w_f, e, bytes); UH_ERR_DOMAIN
 * (n_branches < 1, n_cand < 1, d < 1); UH_ERR_UNSUPPORTED (n_branches > 8); UH_ERR_DIM
 * (branches with different num_seqs, or a sequence with fewer than n_cand rows, checked on
 * the host offsets); UH_ERR_SHAPE (bf16 with
 * d % 64 != 0); UH_ERR_ALIGNMENT (pointers not 16-byte aligned, ld * elem not a multiple of
 * 16 bytes); UH_ERR_WORKSPACE.  B = 0 is a no-op. */
UH_API uh_status uh_mot_fuse_fwd(int32_t n_branches, const uh_mot_branch* branches, int32_t n_cand, int32_t d,
                                 uh_dtype dtype, const void* w_f, const float* b_f, void* e,
                                 void* ws, size_t ws_bytes, void* stream);

/* Backward of uh_mot_fuse_fwd.  de: [C, d] (row stride d, dtype).  dw_f: fp32 [n_branches d, d],
 * db_f: fp32 [d] or NULL; accumulate = 0 overwrites them, 1 adds into them.  dx: host array of
 * n_branches device pointers, dx[k] [T_k, d] with row stride ld_dx[k] (host array), dtype;
 * every row is written (zero outside the candidate rows).  Errors as uh_mot_fuse_fwd, plus
 * UH_ERR_NULL for de, dw_f, dx, ld_dx or a dx[k]. */
UH_API uh_status uh_mot_fuse_bwd(int32_t n_branches, const uh_mot_branch* branches, int32_t n_cand, int32_t d,
                                 uh_dtype dtype, const void* w_f, const void* de, float* dw_f, float* db_f,
                                 int accumulate, void* const* dx, const int64_t* ld_dx,
                                 void* ws, size_t ws_bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* UHSTU_MOT_H */
