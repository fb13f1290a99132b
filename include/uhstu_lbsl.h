/*
 * uhstu_lbsl.h — NEXT-3 of libuhstu: Load-Balanced Stochastic Length (LBSL),
 * arXiv 2602.16986 §4.1 and Algorithm 1 (App. C).
 *
 * LBSL runs per rank between the data loader and the model: it decides, for each
 * example u of the rank's batch, whether the user history is kept whole or sampled
 * down to l_SL tokens, so that the rank's load sum_u n_u^gamma tracks a
 * target l_bar shared by all ranks.  The per-rank decisions are host code (a batch is
 * b ~ 32 lengths); the token gather that applies them is a device kernel.  The
 * target's all-reduce (Alg. 1 lines 22-27) is the caller's (torch.distributed), as is
 * the step counter and the l_r accumulator (see paper_2602_16986_b200/lbsl.py).
 *
 * Readings: R21 StandardSL keeps a user with n_u > l_SL whole with
 * probability (l_SL/n_u)^2 and otherwise samples a uniformly random order-preserving
 * subset of l_SL positions; R22 SLWeight = that keep probability and the
 * "pre-truncation proxy" load = the expected StandardSL load; R23 recalibration after
 * warm-up only; R24 weighted permutation by exponential keys log(r_u)/p_u; R25 the
 * greedy baseline is sum_u min(n_u, l_SL)^gamma; R26 users outside U_r are sampled.
 *
 * Random numbers: a counter-based generator, r = ((h >> 11) + 0.5) * 2^-53 with
 * h = SplitMix64-finaliser chain over (seed, rank, step, stream, idx): stream 0 = the
 * StandardSL choice of user u (idx u), 1 = the permutation key of u (idx u), 2 = the
 * position draws of u (idx (u << 32) | j).  Decisions are therefore a pure function of
 * (lengths, parameters, l_bar, seed, rank, step): reproducible and rank-independent.
 *
 * Conventions of uhstu.h: caller-owned memory, uh_status returns, every check before
 * any side effect.  Host pointers are marked _host, device pointers _dev.
 */
#ifndef UHSTU_LBSL_H
#define UHSTU_LBSL_H
#include "uhstu.h"
#ifdef __cplusplus
extern "C" {
#endif

#define UH_LBSL_TRUNCATED 0  /* sampled down to l_SL positions                        */
#define UH_LBSL_KEPT_BY_SL 1 /* kept whole: n_u <= l_SL, or StandardSL's keep draw       */
#define UH_LBSL_UNSAMPLED 2  /* kept whole: member of the greedy set U_r (Alg. 1 l.14)  */

/* Alg. 1 lines 4-20 for one rank and one step t.
 * lengths_host[b]: raw history lengths n_u >= 0.  ell_sl >= 1 (l_SL), gamma > 0,
 * ell_bar: the current target load; steady = 0 (t <= T_warm: StandardSL on every user,
 * line 7) or 1 (greedy fill, lines 9-18).  Outputs (host, caller-owned):
 * decision_host[b] (UH_LBSL_*), new_len_host[b] (realized lengths), and
 * *proxy_load_host = StandardSL_Loads(B_r) (line 5, the caller adds it to l_r).
 * Sums run in index order in fp64.  Errors: UH_ERR_DOMAIN (b < 0, n_u < 0, ell_sl < 1,
 * gamma <= 0, steady not 0/1), UH_ERR_NULL. */
UH_API uh_status uh_lbsl_select(const int32_t* lengths_host, int32_t b, int32_t ell_sl, double gamma,
                                double ell_bar, int32_t steady, uint64_t seed, int32_t rank, int64_t step,
                                int32_t* decision_host, int32_t* new_len_host, double* proxy_load_host);

/* R21's subset for a sampled user u: tau strictly increasing positions of [0, n)
 * (Knuth's selection sampling with the stream-2 draws of (seed, rank, step, u)) into
 * idx_host[tau].  0 <= tau <= n, else UH_ERR_DOMAIN; u in [0, 2^31). */
UH_API uh_status uh_lbsl_subset(int32_t n, int32_t tau, uint64_t seed, int32_t rank, int64_t step, int32_t u,
                                int32_t* idx_host);

/* Rows of a whole LBSL step: for the jagged batch with host offsets off_host[b+1]
 * (rows of user u are [off[u], off[u+1]), n_u = off[u+1] - off[u]) and the decisions
 * of uh_lbsl_select, writes the source row of every kept token, users in order,
 * positions ascending, into rows_host[sum new_len] and the new offsets into
 * new_off_host[b+1].  Truncated users take uh_lbsl_subset's positions.
 * Errors: UH_ERR_DIM (offsets not non-decreasing, new_len inconsistent), UH_ERR_NULL. */
UH_API uh_status uh_lbsl_rows(const int32_t* off_host, int32_t b, const int32_t* decision_host,
                              const int32_t* new_len_host, uint64_t seed, int32_t rank, int64_t step,
                              int32_t* rows_host, int32_t* new_off_host);

/* Device row gather applying the step: y[i, :] = x[rows_dev[i], :] for i < n_rows.
 * x: [*, width] elements of elem_bytes bytes with row stride ld_x, y: [n_rows, width]
 * with stride ld_y (elements).  x, y 16-byte aligned, width*elem_bytes, ld_x*elem_bytes
 * and ld_y*elem_bytes multiples of 16 (else UH_ERR_ALIGNMENT); row ids are trusted
 * (0 <= rows_dev[i] < rows of x).  One warp per row, 16-byte vector copies; HBM bound.
 * n_rows = 0 is a no-op. */
UH_API uh_status uh_gather_rows(const int32_t* rows_dev, int64_t n_rows, const void* x, int64_t ld_x, int64_t width,
                                int32_t elem_bytes, void* y, int64_t ld_y, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* UHSTU_LBSL_H */
