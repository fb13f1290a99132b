/*
 * ORACLE — test infrastructure only.
 *
 * Plain, slow, fp64 CPU implementation of the jagged semi-local HSTU
 * attention (ULTRA-HSTU, arXiv 2602.16986).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header or constant with the CUDA path
 * (paper_2602_16986_b200/csrc), and the CUDA path never calls it.
 *
 * What it computes (PAPER.md = /root/reference/PAPER.md, "P:n" = line n):
 *   Eq. 3 (§3):          A = (phi2(Q K^T) (.) M) V, phi2 = SiLU, no softmax.
 *   Causal mask (§4.2.1) and the SLA mask (§4.2.1 eq. "M_ij"),
 *   read in time-ascending (q,k) form (readings R1-R4):
 *       allowed(q,k)  <=>  k <= q  and  ( q-k <= K1  or  k < K2 ).
 *   1/N normalisation (R5), score scale alpha (R6) and the relative
 *   position/time bias rab (R7) are DESIGN.md readings, not paper text:
 *       s(q,k) = alpha <Q_q, K_k> + pos_w[min(q-k, P-1)] + ts_w[bkt(t_q - t_k)]
 *       bkt(D) = min(NB-1, floor(log2(max(D,1))))        (exact on integers)
 *       A_q    = sum_{k allowed} silu(s)/N * V_k
 *   Backward (Listing 1, "attention_backward(dattn, q, k, v)"), the
 *   exact chain rule of the forward above:
 *       p = silu(s)/N;  dV_k += p dA_q;  dp = <dA_q, V_k>;
 *       ds = dp * silu'(s)/N,  silu'(s) = sig(s) (1 + s (1 - sig(s)));
 *       dQ_q += alpha ds K_k;  dK_k += alpha ds Q_q;  dpos[..] += ds;  dts[..] += ds.
 *
 * The loops visit ONLY allowed pairs ("work is Theta(mask_nnz*d_h)")
 * and count them in *work.  No blocking, no fusion, no reordering.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* SLA predicate, P:140-146 read as (q,k) with k <= q (R1), inclusive window (R2),
 * global prefix k < K2 (R3).  K1 < 0 means "full causal" (no window limit). */
int orc_mask_allows(int64_t q, int64_t k, int64_t K1, int64_t K2) {
    if (k < 0 || q < 0 || k > q) return 0;
    if (K1 < 0) return 1;
    if (q - k <= K1) return 1;
    if (k < K2) return 1;
    return 0;
}

/* number of allowed (q,k) pairs of a length-L sequence, by enumeration */
int64_t orc_mask_nnz(int64_t L, int64_t K1, int64_t K2) {
    int64_t n = 0;
    for (int64_t q = 0; q < L; ++q)
        for (int64_t k = 0; k <= q; ++k) n += orc_mask_allows(q, k, K1, K2);
    return n;
}

static double silu(double x) { return x / (1.0 + exp(-x)); }
static double sigm(double x) { return 1.0 / (1.0 + exp(-x)); }

/* floor(log2(max(D,1))) computed on integers, then clamped to NB-1 (R7) */
static int64_t time_bucket(int64_t D, int64_t NB) {
    if (D < 1) D = 1;
    int64_t b = 0;
    while ((D >> 1) > 0) { D >>= 1; ++b; }
    return b < NB - 1 ? b : NB - 1;
}

static int64_t pos_index(int64_t dq, int64_t P) { return dq < P - 1 ? dq : P - 1; }

/* score s(q,k) of head h; q,k are absolute token rows, p,pk positions in the sequence */
static double score(const double* Q, const double* K, int64_t ld, int64_t col0, int dh,
                    int64_t rq, int64_t rk, int64_t p, int64_t pk, double alpha,
                    const double* pos_w, int64_t P, const double* ts_w, int64_t NB,
                    const int64_t* t) {
    double acc = 0.0;
    for (int c = 0; c < dh; ++c) acc += Q[rq * ld + col0 + c] * K[rk * ld + col0 + c];
    double s = alpha * acc;
    if (pos_w) s += pos_w[pos_index(p - pk, P)];
    if (ts_w) s += ts_w[time_bucket(t[rq] - t[rk], NB)];
    return s;
}

/*
 * Forward.  Layout: row r of Q/K/V holds all heads; head h occupies columns
 * [h*dh, (h+1)*dh) of the row; row stride ld (elements).  A has stride ldA.
 * offsets[B+1] are the jagged sequence offsets (P:77 X_i in R^{L_i x d}).
 * K1 < 0 selects full causal.  pos_w (length P) / ts_w (length NB) may be NULL.
 */
void orc_attn_fwd(int B, const int32_t* offsets, int H, int dh,
                  const double* Q, const double* K, const double* V, int64_t ld,
                  int64_t K1, int64_t K2, double alpha, double N,
                  const double* pos_w, int64_t P, const double* ts_w, int64_t NB,
                  const int64_t* t, double* A, int64_t ldA, int64_t* work) {
    int64_t total_work = 0;
#pragma omp parallel for collapse(2) schedule(dynamic) reduction(+ : total_work)
    for (int b = 0; b < B; ++b) {
        for (int h = 0; h < H; ++h) {
            int64_t o = offsets[b], L = offsets[b + 1] - offsets[b];
            int64_t col0 = (int64_t)h * dh;
            double* acc = (double*)calloc((size_t)dh, sizeof(double));
            for (int64_t p = 0; p < L; ++p) {
                memset(acc, 0, sizeof(double) * (size_t)dh);
                for (int64_t pk = 0; pk <= p; ++pk) {
                    if (!orc_mask_allows(p, pk, K1, K2)) continue;
                    ++total_work;
                    double s = score(Q, K, ld, col0, dh, o + p, o + pk, p, pk, alpha,
                                     pos_w, P, ts_w, NB, t);
                    double w = silu(s) / N;
                    for (int c = 0; c < dh; ++c) acc[c] += w * V[(o + pk) * ld + col0 + c];
                }
                for (int c = 0; c < dh; ++c) A[(o + p) * ldA + col0 + c] = acc[c];
            }
            free(acc);
        }
    }
    if (work) *work = total_work;
}

/*
 * Backward of orc_attn_fwd for upstream gradient dA (stride ldA).  Writes
 * dQ, dK, dV (stride ldG, overwritten) and ACCUMULATES into dpos[P] / dts[NB]
 * (caller zeroes them).  dpos/dts may be NULL when the matching table is NULL.
 * dpos_abs / dts_abs (nullable) accumulate |ds| per entry: the sum of the absolute
 * terms, the scale of the summation error bound for these cancelling sums (reading R15b).
 */
void orc_attn_bwd(int B, const int32_t* offsets, int H, int dh,
                  const double* Q, const double* K, const double* V, int64_t ld,
                  const double* dA, int64_t ldA,
                  int64_t K1, int64_t K2, double alpha, double N,
                  const double* pos_w, int64_t P, const double* ts_w, int64_t NB,
                  const int64_t* t,
                  double* dQ, double* dK, double* dV, int64_t ldG,
                  double* dpos, double* dts, double* dpos_abs, double* dts_abs, int64_t* work) {
    int nthr = 1;
#ifdef _OPENMP
    nthr = omp_get_max_threads();
#endif
    double* dpos_t = (pos_w && dpos) ? (double*)calloc((size_t)nthr * (size_t)P, sizeof(double)) : NULL;
    double* dts_t = (ts_w && dts) ? (double*)calloc((size_t)nthr * (size_t)NB, sizeof(double)) : NULL;
    double* dpos_at = (pos_w && dpos_abs) ? (double*)calloc((size_t)nthr * (size_t)P, sizeof(double)) : NULL;
    double* dts_at = (ts_w && dts_abs) ? (double*)calloc((size_t)nthr * (size_t)NB, sizeof(double)) : NULL;
    int64_t total_work = 0;

    /* zero the gradient rows of every sequence (only real rows are touched) */
    for (int b = 0; b < B; ++b)
        for (int64_t r = offsets[b]; r < offsets[b + 1]; ++r)
            for (int64_t c = 0; c < (int64_t)H * dh; ++c) {
                dQ[r * ldG + c] = 0.0; dK[r * ldG + c] = 0.0; dV[r * ldG + c] = 0.0;
            }

#pragma omp parallel for collapse(2) schedule(dynamic) reduction(+ : total_work)
    for (int b = 0; b < B; ++b) {
        for (int h = 0; h < H; ++h) {
            int tid = 0;
#ifdef _OPENMP
            tid = omp_get_thread_num();
#endif
            int64_t o = offsets[b], L = offsets[b + 1] - offsets[b];
            int64_t col0 = (int64_t)h * dh;
            for (int64_t p = 0; p < L; ++p) {
                int64_t rq = o + p;
                for (int64_t pk = 0; pk <= p; ++pk) {
                    if (!orc_mask_allows(p, pk, K1, K2)) continue;
                    ++total_work;
                    int64_t rk = o + pk;
                    double s = score(Q, K, ld, col0, dh, rq, rk, p, pk, alpha,
                                     pos_w, P, ts_w, NB, t);
                    double pw = silu(s) / N;
                    double dp = 0.0;
                    for (int c = 0; c < dh; ++c) {
                        dV[rk * ldG + col0 + c] += pw * dA[rq * ldA + col0 + c];
                        dp += dA[rq * ldA + col0 + c] * V[rk * ld + col0 + c];
                    }
                    double sg = sigm(s);
                    double ds = dp * sg * (1.0 + s * (1.0 - sg)) / N;
                    for (int c = 0; c < dh; ++c) {
                        dQ[rq * ldG + col0 + c] += alpha * ds * K[rk * ld + col0 + c];
                        dK[rk * ldG + col0 + c] += alpha * ds * Q[rq * ld + col0 + c];
                    }
                    if (dpos_t) dpos_t[(size_t)tid * P + pos_index(p - pk, P)] += ds;
                    if (dts_t) dts_t[(size_t)tid * NB + time_bucket(t[rq] - t[rk], NB)] += ds;
                    if (dpos_at) dpos_at[(size_t)tid * P + pos_index(p - pk, P)] += fabs(ds);
                    if (dts_at) dts_at[(size_t)tid * NB + time_bucket(t[rq] - t[rk], NB)] += fabs(ds);
                }
            }
        }
    }
    for (int i = 0; i < nthr; ++i) {
        if (dpos_t) for (int64_t j = 0; j < P; ++j) dpos[j] += dpos_t[(size_t)i * P + j];
        if (dts_t) for (int64_t j = 0; j < NB; ++j) dts[j] += dts_t[(size_t)i * NB + j];
        if (dpos_at) for (int64_t j = 0; j < P; ++j) dpos_abs[j] += dpos_at[(size_t)i * P + j];
        if (dts_at) for (int64_t j = 0; j < NB; ++j) dts_abs[j] += dts_at[(size_t)i * NB + j];
    }
    free(dpos_t);
    free(dts_t);
    free(dpos_at);
    free(dts_at);
    if (work) *work = total_work;
}

int orc_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
