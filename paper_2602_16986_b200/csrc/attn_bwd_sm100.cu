// attn_bwd_sm100.cu — jagged semi-local HSTU attention backward on tcgen05.
//
// Listing 1's "dq, dk, dv = attention_backward(dattn, q, k, v)" for the
// forward of attn_fwd_sm100.cu (Eq. 3; SLA P:140-146; R5-R7):
//     p = silu(s)/N, ds = dP * silu'(s)/N, dP = dA V^T, s = alpha Q K^T + rab
//     dV = P^T dA,  dK = alpha dS^T Q,  dQ = alpha dS K,  d rab = scatter-sum of ds.
// One kernel, fb::attn_bwd_fused_sm100 (a key-major pass): per 128-key tile (K, V resident in
// shared memory), over the 64-query steps that see it: S^T = K Q^T and dP^T = V dA^T (SS);
// the P/dS warpgroups (warps 4-11) write P^T, dS^T (bf16) over the consumed TMEM columns and
// dS^T to shared memory, and sum d time_bias; dV += P^T dA, dK += dS^T Q (TS);
// dQ^T = K^T dS^T (SS) over the consumed S^T columns, read by the two dQ warpgroups (warps
// 12-19) and TMA-added into an fp32 [T, H dh] accumulator, which dq_finish_k scales and
// gates into dQ; the dQ warpgroups also sum d pos_bias from the dS^T tile.
// TMEM buffers are reused in tensor-pipe order (an MMA issued after another by the same
// thread executes after it).
// Gradients are multiplied by optional gates (silu'(h), the layer's fused
// "silu_backward") and written straight into their slices of dH (no
// concat).
#include <climits>
#include <cstdlib>
#include <cstring>

#include "attn_common.cuh"
#include "internal.h"

namespace uh {
namespace {

constexpr int DH = 128;

__device__ __forceinline__ void store_out_row64(void* base, int64_t ld, int64_t row, int col, const float* v,
                                                const void* gate, int64_t ldg, float scale) {
    float w[64];
#pragma unroll
    for (int c = 0; c < 64; ++c) w[c] = v[c] * scale;
    const bool v8 = ((reinterpret_cast<uintptr_t>(base) | (uintptr_t)(ld * 2) |
                      (gate ? (reinterpret_cast<uintptr_t>(gate) | (uintptr_t)(ldg * 2)) : 0)) & 31) == 0;
    if (gate) {
        const __nv_bfloat16* gp = reinterpret_cast<const __nv_bfloat16*>(gate) + row * ldg + col;
#pragma unroll
        for (int ch = 0; ch < 8; ch += 2) {
            uint32_t gw[8];
            if (v8) {
                asm volatile("ld.global.nc.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                             : "=r"(gw[0]), "=r"(gw[1]), "=r"(gw[2]), "=r"(gw[3]), "=r"(gw[4]), "=r"(gw[5]),
                               "=r"(gw[6]), "=r"(gw[7]) : "l"(gp + ch * 8));
            } else {
                const uint4 a0 = __ldg(reinterpret_cast<const uint4*>(gp + ch * 8));
                const uint4 a1 = __ldg(reinterpret_cast<const uint4*>(gp + ch * 8 + 8));
                gw[0] = a0.x; gw[1] = a0.y; gw[2] = a0.z; gw[3] = a0.w;
                gw[4] = a1.x; gw[5] = a1.y; gw[6] = a1.z; gw[7] = a1.w;
            }
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const float2 f = unpack_bf16x2(gw[e]);
                w[ch * 8 + 2 * e] *= f.x;
                w[ch * 8 + 2 * e + 1] *= f.y;
            }
        }
    }
    __nv_bfloat16* op = reinterpret_cast<__nv_bfloat16*>(base) + row * ld + col;
#pragma unroll
    for (int ch = 0; ch < 8; ch += 2) {
        uint32_t p[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) p[e] = pack_bf16(w[ch * 8 + 2 * e], w[ch * 8 + 2 * e + 1]);
        if (v8) {
            asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(op + ch * 8), "r"(p[0]), "r"(p[1]),
                         "r"(p[2]), "r"(p[3]), "r"(p[4]), "r"(p[5]), "r"(p[6]), "r"(p[7]) : "memory");
        } else {
            *reinterpret_cast<uint4*>(op + ch * 8) = make_uint4(p[0], p[1], p[2], p[3]);
            *reinterpret_cast<uint4*>(op + ch * 8 + 8) = make_uint4(p[4], p[5], p[6], p[7]);
        }
    }
}

// sum of 32 fp32 values as a tree of packed FADD2
__device__ __forceinline__ float sum32_f2(const float* v) {
    uint64_t x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fadd2(f2_pack(v[4 * i], v[4 * i + 1]), f2_pack(v[4 * i + 2], v[4 * i + 3]));
#pragma unroll
    for (int i = 0; i < 4; ++i) x[i] = fadd2(x[i], x[i + 4]);
    x[0] = fadd2(x[0], x[2]); x[1] = fadd2(x[1], x[3]);
    const float2 r = f2_unpack(fadd2(x[0], x[1]));
    return r.x + r.y;
}

// ============================================================================ fused kernel
// One pass per 128-key tile computes dV, dK and the dQ partials of every visible 64-query
// step: dQ^T = K^T dS^T (SS, M = dh, N = 64) lands in the TMEM columns of the consumed
// S^T, is read by a fourth warpgroup and added into an fp32 [T, H dh] buffer with TMA
// reductions (in L2: the schedule's consecutive key tiles keep the touched query rows
// L2-resident).  S, P and dP are computed once instead of once per kernel.  The rab
// gradients: d time_bias in the P/dS epilogue from the fp32 dS (per-lane bucket runs,
// shared atomics), d pos_bias in the dQ warpgroup from the dS^T tile in shared memory
// (skewed-shuffle diagonal sums, one global reduction per diagonal and warp), any P.
namespace fb {
#if UH_TRACE == 3   // per-step timeline of CTA 0 (tools/trace_fused.py)
#define TRACE_FB(ev, sc) do { if (lane == 0) TRACE((ev) * 1024 + ((sc) & 1023)); } while (0)
#else
#define TRACE_FB(ev, sc) do { } while (0)
#endif
constexpr int BM = 128, BN = 64;          // 128 keys (MMA M), 64 queries per step
constexpr int KT = BM * DH * 2;           // K / V tile (32 KB: 2 x 16 KB blocks of [128 rows x 128 B])
constexpr int QT = BN * DH * 2;           // Q / dA tile (16 KB: 2 x 8 KB blocks of [64 rows x 128 B])
constexpr int STAGES = 3;                 // (Q, dA) ring
constexpr int DS_BYTES = BM * BN * 2;     // dS^T [128 keys][64 queries] bf16, one SW128 block
constexpr int STG_BYTES = 32 * 32 * 4;    // per dQ warp: [32 queries][32 dh] fp32 box
constexpr int THREADS = 640;              // w0 TMA, w1 MMA (S/dP), w2 TMEM alloc, w3 MMA (dV/dK/dQ),
                                          // w4-11 P/dS epilogue, w12-15 dQ + d rab
constexpr int S_COL = 0, DP_COL = 128, DV_COL = 256, DK_COL = 384;
constexpr int DTS_LANES = 16;             // d time_bias partials [32 buckets][16 lane slots] (2-way at most)
constexpr int SMEM_DATA = 2 * KT + STAGES * 2 * QT + 2 * DS_BYTES + 8 * STG_BYTES + 32 * 4 + 32 * DTS_LANES * 4 + 512;
// registers per thread after setmaxnreg (640 threads start at 96): control warps / P-dS / dQ warpgroups.
// An increase is served only from what the CTA's own decreases released.
constexpr int REG_LAUNCH = 96, REG_CTRL = 48, REG_PDS = 136, REG_DQ = 80;
static_assert(128 * (REG_LAUNCH - REG_CTRL) + 256 * (REG_LAUNCH - REG_DQ) >= 256 * (REG_PDS - REG_LAUNCH),
              "setmaxnreg: the P/dS increase must fit in the released registers");
// dynamic shared memory starts 1024-byte aligned (the CTA's first 1 KB is reserved by the
// hardware); the kernel traps otherwise, since the SW128 tiles need it
constexpr int SMEM = SMEM_DATA;
static_assert(SMEM <= 232448, "fused bwd shared memory");

struct __align__(8) Bars {
    uint64_t kv_full, kv_empty;
    uint64_t qa_full[STAGES], qa_empty[STAGES];
    uint64_t s_full[2], p_full[2];
    uint64_t dq_full[2];    // dQ^T(i) in the S columns of buffer i & 1
    uint64_t s_free[2];     // ... read by the dQ warps: the next S^T may overwrite them
    uint64_t ds_free[2];    // dS^T shared buffer read by the dQ MMA and the d pos_bias reduction
    uint64_t acc_full, acc_empty;
    ItemRing ring;
    uint32_t tmem;
};

__device__ __forceinline__ int n_qtiles(int k0, int L, int K1, int K2) {
    const int qe = query_end(k0, BM, L, K1, K2);
    return (qe + BN - 1) / BN - k0 / BN;
}

__global__ void __launch_bounds__(THREADS, 1)
attn_bwd_fused_sm100(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                     const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmdA,
                     const __grid_constant__ CUtensorMap tmDQ, AttnArgs a) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    if (smem_u32(smem_raw) & 1023) __trap();
    uint8_t* smem = smem_raw;
    uint8_t* sK = smem;                                   // K 32 KB | V 32 KB
    uint8_t* sV = smem + KT;
    uint8_t* sQA = smem + 2 * KT;                         // [STAGES] x (Q 16 KB | dA 16 KB)
    uint8_t* sDS = sQA + STAGES * 2 * QT;                 // [2] x dS^T
    float* sDQ = reinterpret_cast<float*>(sDS + 2 * DS_BYTES);   // [8 warps] x [32][32] fp32
    float* ts_s = sDQ + 8 * STG_BYTES / 4;                // time_bias / 2 [32]
    float* dts_s = ts_s + 32;                             // d time_bias partials [32 buckets][DTS_LANES]
    Bars* bars = reinterpret_cast<Bars*>(dts_s + 32 * DTS_LANES);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    TRACE_SETUP();

    if (threadIdx.x == 0) {
        mbar_init(&bars->kv_full, 1); mbar_init(&bars->kv_empty, 1);
        for (int i = 0; i < STAGES; ++i) { mbar_init(&bars->qa_full[i], 1); mbar_init(&bars->qa_empty[i], 1); }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&bars->s_full[i], 1); mbar_init(&bars->p_full[i], 8); mbar_init(&bars->dq_full[i], 1);
            mbar_init(&bars->s_free[i], 8); mbar_init(&bars->ds_free[i], 8);
        }
        mbar_init(&bars->acc_full, 1); mbar_init(&bars->acc_empty, 8);
        ring_init(&bars->ring, 18);  // MMA warps 1, 3 + 8 P/dS warps + 8 dQ warps
        fence_barrier_init();
    }
    stage_ts(a, ts_s);
    for (int i = threadIdx.x; i < 32 * DTS_LANES; i += THREADS) dts_s[i] = 0.f;
    if (warp == 2) tmem_alloc<512>(&bars->tmem);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = bars->tmem;
    // the register file is rebalanced by warpgroup at the top of every role (setmaxnreg: all warps
    // of a warpgroup execute the same one): control warps REG_CTRL, P/dS REG_PDS, dQ REG_DQ
    if (warp < 4) {
        // control warpgroup: TMA producer (warp 0), MMA issuers (warps 1, 3), TMEM allocator (2)
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(REG_CTRL));
    if (warp == 0) {
        // ============================================================ producer
        if (lane == 0) {
            int qc = 0, ki = 0;
            for (;; ++ki) {
                const int w = ring_claim_publish(&bars->ring, ki, a.counter, a.n_items);
                if (w < 0) break;
                const WorkItem it = a.items[w];
                check_item(a, it, BM);
                const int k0 = it.tile * BM, h = it.head & 0xFFFF;
                const int n = n_qtiles(k0, it.seq_len, a.K1, a.K2);
                mbar_wait_sleep(&bars->kv_empty, (ki & 1) ^ 1);
                mbar_arrive_expect_tx(&bars->kv_full, 2 * KT);
                tma_load_2d(sK, &tmK, &bars->kv_full, h * DH, it.seq_start + k0);
                tma_load_2d(sK + KT / 2, &tmK, &bars->kv_full, h * DH + 64, it.seq_start + k0);
                tma_load_2d(sV, &tmV, &bars->kv_full, h * DH, it.seq_start + k0);
                tma_load_2d(sV + KT / 2, &tmV, &bars->kv_full, h * DH + 64, it.seq_start + k0);
                for (int i = 0; i < n; ++i) {
                    const int row = it.seq_start + (k0 / BN + i) * BN;
                    const int s = qc % STAGES;
                    uint8_t* st = sQA + s * 2 * QT;
                    mbar_wait_sleep(&bars->qa_empty[s], ((qc / STAGES) & 1) ^ 1);
                    TRACE_FB(7, qc);
                    mbar_arrive_expect_tx(&bars->qa_full[s], 2 * QT);
                    tma_load_2d(st, &tmQ, &bars->qa_full[s], h * DH, row);
                    tma_load_2d(st + QT / 2, &tmQ, &bars->qa_full[s], h * DH + 64, row);
                    tma_load_2d(st + QT, &tmdA, &bars->qa_full[s], h * DH, row);
                    tma_load_2d(st + QT + QT / 2, &tmdA, &bars->qa_full[s], h * DH + 64, row);
                    ++qc;
                }
            }
        }
    } else if (warp == 1 || warp == 3) {
        // ============================================================ MMA issuers
        // warp 1: S^T(i) = K Q_i^T, dP^T(i) = V dA_i^T into buffer i & 1, once the dQ warps have
        // read dQ^T(i - 2) from it.  warp 3: dV += P^T dA, dK += dS^T Q (TMEM A operands), then
        // dQ^T(i) = K^T dS^T (both from shared memory) over the consumed S^T columns — issued
        // after the dV MMA that reads P^T there (one warp, tensor-pipe order).
        constexpr uint32_t idesc_s = make_idesc_bf16(BM, BN, false, false);   // [K|V] x [Q|dA]^T (both K-major)
        constexpr uint32_t idesc_a = make_idesc_bf16(BM, DH, false, true);    // [P^T|dS^T](TMEM) x [dA|Q] (MN-major)
        constexpr uint32_t idesc_q = make_idesc_bf16(DH, BN, true, true);     // K^T (MN-major) x dS^T (MN-major)
        int ki = 0, sc = 0;
        if (warp == 1) {
            const uint64_t kv_k = make_sw128_desc(smem_u32(sK), 16, 1024);       // K / V K-major (A)
            const uint64_t q_k = make_sw128_desc(smem_u32(sQA), 16, 1024);       // Q / dA K-major (B)
            int st_s = 0, ph_s = 0;
            for (;; ++ki) {
                const int w = ring_take(&bars->ring, ki, lane);
                if (w < 0) break;
                const WorkItem it = a.items[w];
                check_item(a, it, BM);
                const int n = n_qtiles(it.tile * BM, it.seq_len, a.K1, a.K2);
                const uint64_t dk = kv_k, dv = dk + (KT >> 4);
                mbar_wait(&bars->kv_full, ki & 1);
                mbar_wait(&bars->qa_full[st_s], ph_s);
                mbar_wait(&bars->s_free[sc & 1], ((sc >> 1) - 1) & 1);   // (first steps: parity 1 of a fresh barrier passes)
                for (int i = 0; i < n; ++i, ++sc) {
                    const int sb = sc & 1;
                    tc_fence_after();
                    const int nst = st_s + 1 == STAGES ? 0 : st_s + 1, nph = st_s + 1 == STAGES ? ph_s ^ 1 : ph_s;
                    const uint32_t qa_a = smem_u32(&bars->qa_full[nst]), sf_a = smem_u32(&bars->s_free[sb ^ 1]);
                    const uint32_t sf_p = (((sc + 1) >> 1) - 1) & 1;
                    const bool r1 = mbar_test(qa_a, nph), r2 = mbar_test(sf_a, sf_p);
                    const uint64_t dq = q_k + ((uint32_t)(st_s * 2 * QT) >> 4), dda = dq + (QT >> 4);
                    const uint32_t d_s = tmem + S_COL + sb * BN, d_p = tmem + DP_COL + sb * BN;
                    TRACE_FB(0, sc);
                    if (elect_one()) {
#pragma unroll
                        for (int kk = 0; kk < DH / 16; ++kk) {
                            const uint32_t oa = ((kk >> 2) * (KT / 2) + (kk & 3) * 32) >> 4;
                            const uint32_t ob = ((kk >> 2) * (QT / 2) + (kk & 3) * 32) >> 4;
                            umma_ss(d_s, dk + oa, dq + ob, idesc_s, kk > 0 ? 1u : 0u);
                            umma_ss(d_p, dv + oa, dda + ob, idesc_s, kk > 0 ? 1u : 0u);
                        }
                        umma_commit(&bars->s_full[sb]);
                    }
                    __syncwarp();
                    st_s = nst; ph_s = nph;
                    if (i + 1 < n) {
                        if (!r1) mbar_wait_addr(qa_a, nph);
                        if (!r2) mbar_wait_addr(sf_a, sf_p);
                    }
                }
            }
        } else {
            const uint64_t q_mn = make_sw128_desc(smem_u32(sQA), QT / 2, 1024);  // Q / dA MN-major (B)
            const uint64_t kt_mn = make_sw128_desc(smem_u32(sK), KT / 2, 1024);  // K^T: M = dh over 2 blocks
            const uint64_t ds_mn = make_sw128_desc(smem_u32(sDS), DS_BYTES, 1024);  // dS^T: N = 64 queries
            int st_a = 0;
            for (;; ++ki) {
                const int w = ring_take(&bars->ring, ki, lane);
                if (w < 0) break;
                const WorkItem it = a.items[w];
                check_item(a, it, BM);
                const int n = n_qtiles(it.tile * BM, it.seq_len, a.K1, a.K2);
                mbar_wait(&bars->acc_empty, (ki & 1) ^ 1);
                mbar_wait(&bars->p_full[sc & 1], (sc >> 1) & 1);
                for (int i = 0; i < n; ++i, ++sc) {
                    const int pb = sc & 1;
                    tc_fence_after();
                    const uint32_t pf_a = smem_u32(&bars->p_full[pb ^ 1]), pf_p = ((sc + 1) >> 1) & 1;
                    const bool r = mbar_test(pf_a, pf_p);   // step i+1's P^T / dS^T
                    const uint64_t dq = q_mn + ((uint32_t)(st_a * 2 * QT) >> 4), dda = dq + (QT >> 4);
                    const uint32_t a_p = tmem + S_COL + pb * BN, a_d = tmem + DP_COL + pb * BN;
                    const uint64_t dsd = ds_mn + ((uint32_t)(pb * DS_BYTES) >> 4);
                    TRACE_FB(1, sc);
                    if (elect_one()) {
#pragma unroll
                        for (int kk = 0; kk < BN / 16; ++kk) {
                            // queries [16 kk, 16 kk + 16): packed by warpgroup kk / 2 at column 32 (kk / 2) + 8 (kk % 2)
                            const uint32_t ca = (kk >> 1) * 32 + (kk & 1) * 8;
                            const uint32_t acc = (i > 0 || kk > 0) ? 1u : 0u;
                            umma_ts(tmem + DV_COL, a_p + ca, dda + kk * (2048 >> 4), idesc_a, acc);
                            umma_ts(tmem + DK_COL, a_d + ca, dq + kk * (2048 >> 4), idesc_a, acc);
                        }
                        umma_commit(&bars->qa_empty[st_a]);
#pragma unroll
                        for (int kk = 0; kk < BM / 16; ++kk)   // keys [16 kk, 16 kk + 16): 16 rows of 128 B
                            umma_ss(a_p, kt_mn + kk * (2048 >> 4), dsd + kk * (2048 >> 4), idesc_q, kk > 0 ? 1u : 0u);
                        umma_commit(&bars->dq_full[pb]);
                        if (i == n - 1) {
                            umma_commit(&bars->acc_full);
                            umma_commit(&bars->kv_empty);   // K (dQ^T) and V (dP^T) read
                        }
                    }
                    tc_fence_before();
                    __syncwarp();
                    if (++st_a == STAGES) st_a = 0;
                    if (i + 1 < n && !r) mbar_wait_addr(pf_a, pf_p);
                }
            }
        }
    }

    } else if (warp < 12) {
        // ============================================================ P / dS epilogue
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(REG_PDS));
        const int wg = (warp - 4) >> 2, wq = warp & 3;
        const int r = wq * 32 + lane;
        const uint32_t lane_base = (uint32_t)(wq * 32) << 16;
        const float ha = 0.5f * a.alpha;
        int sc = 0, ki = 0;
        for (;; ++ki) {
            const int w = ring_take(&bars->ring, ki, lane);
            if (w < 0) break;
            const WorkItem it = a.items[w];
            check_item(a, it, BM);
            const int L = it.seq_len, o = it.seq_start, h = it.head & 0xFFFF;
            const int k0 = it.tile * BM;
            const int n = n_qtiles(k0, L, a.K1, a.K2);
            const int kp = k0 + r;
            const bool kok = kp < L;
            const ChunkCtx cx = make_ctx(a, ts_s, o, L);
            const int32_t tk = (a.ts && kok) ? rel32(__ldg(a.t + o + kp), cx.t0) : 0;
            // d time_bias: buckets are monotone along the key row (sorted timestamps), so the
            // row's dS' values are summed in registers per run of equal bucket and a run is
            // added to the CTA's shared partials only when the bucket changes (slot lane % 16 of
            // the bucket's row: lanes of one flush never share an address)
            float* const dts_l = dts_s + (lane & (DTS_LANES - 1));
            int run_b = 0;
            float run_v = 0.f;
            auto run_add = [&](int b, float v) {
                UH_CHECK(b >= 0 && b < a.NB);
                if (b != run_b) {
                    if (run_v != 0.f) atomicAdd(dts_l + run_b * DTS_LANES, run_v);
                    run_b = b; run_v = 0.f;
                }
                run_v += v;
            };
            for (int i = 0; i < n; ++i, ++sc) {
                const int sb = sc & 1;
                const int qb = (k0 / BN + i) * BN + 32 * wg;   // this warpgroup's 32 queries
                const int32_t tcur = col_time(cx, qb, lane);
                const Chunk ch = k_chunk(cx, kp, kok, tk, qb, tcur);
                mbar_wait_sleep(&bars->s_full[sb], (sc >> 1) & 1);
                __syncwarp();   // tcgen05.ld is .sync.aligned: reconverge after the per-lane wait loop
                if (warp == 4) TRACE_FB(2, sc);
                if (warp == 8) TRACE_FB(4, sc);
                tc_fence_after();
                float sv[32], dp[32];
                tmem_ld32(tmem + lane_base + S_COL + sb * BN + 32 * wg, sv);
                tmem_ld32(tmem + lane_base + DP_COL + sb * BN + 32 * wg, dp);
                tmem_ld_wait();
                float hx[32];
                k_h(cx, ch, tk, sv, hx);
                if (ch.flags & FLAG_M) {          // h = 0 and dP = 0 -> P = dS = 0
                    const uint32_t m = k_vis_bits(cx, kp, kok, qb);
                    apply_vis(hx, m);
                    apply_vis(dp, m);
                }
                uint32_t p2[16], d2[16];
                const uint64_t one2 = f2_pack(1.f, 1.f), neg2 = f2_pack(-1.f, -1.f);
#pragma unroll
                for (int c = 0; c < 16; ++c) {   // fp32 pairs: P = h (1 + t), dS = dP (1 + t)(1 + h (1 - t))
                    const uint64_t H = f2_pack(hx[2 * c], hx[2 * c + 1]);
                    const uint64_t T = f2_pack(tanh_approx(hx[2 * c]), tanh_approx(hx[2 * c + 1]));
                    const uint64_t A1 = fadd2(T, one2);
                    const float2 pv = f2_unpack(fmul2(H, A1));
                    p2[c] = pack_bf16(pv.x, pv.y);
                    const uint64_t W = ffma2(H, ffma2(T, neg2, one2), one2);
                    const float2 dv = f2_unpack(fmul2(fmul2(f2_pack(dp[2 * c], dp[2 * c + 1]), A1), W));
                    // keys beyond L (must not reach dQ) arrive with h = dP = 0 (FLAG_M), so dS = 0
                    d2[c] = pack_bf16(dv.x, dv.y);
                    dp[2 * c] = dv.x;                             // dp now holds the fp32 dS'
                    dp[2 * c + 1] = dv.y;
                }
                // P^T, dS^T -> TMEM over the consumed S^T / dP^T columns (A operands of dV, dK)
                tmem_st16(tmem + lane_base + S_COL + sb * BN + 32 * wg, p2);
                tmem_st16(tmem + lane_base + DP_COL + sb * BN + 32 * wg, d2);
                // dS^T -> shared memory (B operand of dQ^T, input of the d rab reduction)
                mbar_wait(&bars->ds_free[sb], ((sc >> 1) - 1) & 1);
                store_row32_packed(sDS + sb * DS_BYTES, r, 32 * wg, d2);
                fence_proxy_async_smem();
                tmem_st_wait();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&bars->p_full[sb]);
                if (warp == 4) TRACE_FB(3, sc);
                if (a.dts) {   // runs of equal time bucket along the row (FLAG_T1: two, FLAG_T2: per element)
                    if (!(ch.flags & FLAG_T2)) {
                        float tsum = sum32_f2(dp), so = 0.f;
                        if (ch.flags & FLAG_T1) {   // columns [n, 32) are in bucket b_other
                            float m[32];
#pragma unroll
                            for (int j = 0; j < 32; ++j) m[j] = j >= ch.n ? dp[j] : 0.f;
                            so = sum32_f2(m);
                        }
                        run_add(ch.b_base, tsum - so);
                        if (ch.n < 32) run_add(ch.b_other, so);
                    } else {
#pragma unroll
                        for (int j = 0; j < 32; ++j)
                            run_add(bucket32(__shfl_sync(0xffffffffu, ch.tcol, j) - tk, cx.NB), dp[j]);
                    }
                }
            }
            if (run_v != 0.f) atomicAdd(dts_l + run_b * DTS_LANES, run_v);
            mbar_wait_sleep(&bars->acc_full, ki & 1);
            __syncwarp();
            tc_fence_after();
            {   // dV then dK (64 registers at a time under the 512-thread register budget)
                float acc[64];
                tmem_ld32(tmem + lane_base + DV_COL + wg * 64, acc);
                tmem_ld32(tmem + lane_base + DV_COL + wg * 64 + 32, acc + 32);
                tmem_ld_wait();
                UH_CHECK(!kok || o + kp < a.T);
                if (kok) store_out_row64(a.dv, a.ld_grad, o + kp, h * DH + wg * 64, acc, a.gv, a.ld_gate, a.inv_n);
                tmem_ld32(tmem + lane_base + DK_COL + wg * 64, acc);
                tmem_ld32(tmem + lane_base + DK_COL + wg * 64 + 32, acc + 32);
                tmem_ld_wait();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&bars->acc_empty);
                if (kok) store_out_row64(a.dk, a.ld_grad, o + kp, h * DH + wg * 64, acc, a.gk, a.ld_gate, ha * a.inv_n);
            }
        }
        // the CTA's d time_bias partials -> one global atomic per bucket
        __syncwarp();
        named_bar_sync(4, 256);
        const int t = threadIdx.x - 128;
        if (a.dts && t < a.NB) {
            float v = 0.f;
#pragma unroll
            for (int l = 0; l < DTS_LANES; ++l) v += dts_s[t * DTS_LANES + l];
            if (v != 0.f) atomicAdd(a.dts + t, v * (0.5f * a.inv_n));
        }
    } else {
        // ============================================================ dQ + d pos_bias
        // two warpgroups: warpgroup hf takes queries [32 hf, 32 hf + 32) of every step
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(REG_DQ));
        const int wq = warp & 3, hf = (warp - 12) >> 2;
        const int r = wq * 32 + lane;                       // key row of this thread (d pos_bias)
        const uint32_t lane_base = (uint32_t)(wq * 32) << 16;   // TMEM lanes = dh [32 wq, 32 wq + 32)
        float* stg = sDQ + (warp - 12) * (STG_BYTES / 4);
        const float rscale = 0.5f * a.inv_n;                // ds = rscale * ds'
        float far_acc = 0.f;                                // sum of ds' at offsets >= P - 1 (this lane)
        auto emit_pos = [&](int dd, float v) {
            if (dd < 0 || v == 0.f) return;
            if (dd >= a.P - 1) far_acc += v;
            else { UH_CHECK(dd >= 0 && dd < a.P - 1); atomicAdd(a.dpos + dd, v * rscale); }
        };
        int sc = 0, ki = 0;
        for (;; ++ki) {
            const int w = ring_take(&bars->ring, ki, lane);
            if (w < 0) break;
            const WorkItem it = a.items[w];
            check_item(a, it, BM);
            const int L = it.seq_len, o = it.seq_start, h = it.head & 0xFFFF;
            const int k0 = it.tile * BM;
            const int n = n_qtiles(k0, L, a.K1, a.K2);
            for (int i = 0; i < n; ++i, ++sc) {
                const int sb = sc & 1;
                const int qb0 = (k0 / BN + i) * BN;
                mbar_wait_sleep(&bars->dq_full[sb], (sc >> 1) & 1);
                __syncwarp();
                if (warp == 12) TRACE_FB(5, sc);
                tc_fence_after();
                float v[32];
                tmem_ld32(tmem + lane_base + S_COL + sb * BN + 32 * hf, v);
                tmem_ld_wait();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&bars->s_free[sb]);
                // [32 queries][32 dh] box -> TMA add into the fp32 accumulator (rows past L add zeros)
                if (lane == 0) bulk_wait_read0();
                __syncwarp();
#pragma unroll
                for (int q = 0; q < 32; ++q) stg[q * 32 + lane] = v[q];
                fence_proxy_async_smem();
                __syncwarp();
                UH_CHECK(qb0 + 32 * hf < L + BN && h < a.H);
                if (lane == 0) {
                    tma_reduce_add_2d(&tmDQ, stg, h * DH + 32 * wq, o + qb0 + 32 * hf);
                    bulk_commit();
                }
                if (a.dpos) {
                    // d pos_bias[min(q - k, P - 1)] += ds: in this warp's 32 x 32 block of dS^T the
                    // element (row s, column c) sits on diagonal C + c - s; a skewed shuffle (lane m
                    // reads the bf16 pair of columns c, c + 1 from lane (c - m) mod 32, c even) gives
                    // lane m the sums of diagonals C + m (c >= m) and C + m - 32 (c < m), half of them
                    // via lane m - 1 (16 shuffles + 2; the 32-shuffle form: 2.908 -> 2.836 ms): two
                    // global reductions per lane and block; blocks whose offsets all clamp to P - 1
                    // accumulate in a register.
                    const int C = qb0 + 32 * hf - k0 - 32 * wq;
                    if (C + 31 >= 0) {                             // warp-uniform: else strictly upper (masked)
                        mbar_wait(&bars->p_full[sb], (sc >> 1) & 1);   // the P/dS warps' shared stores are visible
                        const uint8_t* row = sDS + sb * DS_BYTES + r * 128;
                        uint32_t d2[16];
#pragma unroll
                        for (int c = 0; c < 4; ++c) {
                            const uint4 u = *reinterpret_cast<const uint4*>(row + (((4 * hf + c) ^ (r & 7)) << 4));
                            d2[4 * c] = u.x; d2[4 * c + 1] = u.y; d2[4 * c + 2] = u.z; d2[4 * c + 3] = u.w;
                        }
                        if (C - 31 >= a.P - 1) {                   // warp-uniform: every offset clamps to P - 1
                            far_acc += sum_packed16(d2);
                        } else {
                            // even columns c: the pair (c, c + 1) of row (c - m) mod 32; element c lies on
                            // lane m's diagonal (C + m, or C + m - 32 when c < m), element c + 1 on lane
                            // m+1's (same wrap condition)
                            uint64_t nw = f2_pack(0.f, 0.f), wr = nw;   // (own, next lane's): c >= m / c < m
#pragma unroll
                            for (int c = 0; c < 32; c += 2) {
                                const float2 u = unpack_bf16x2(__shfl_sync(0xffffffffu, d2[c >> 1], (c - lane) & 31));
                                const uint64_t u2 = f2_pack(u.x, u.y);
                                if (c < lane) wr = fadd2(wr, u2); else nw = fadd2(nw, u2);
                            }
                            const float2 a2 = f2_unpack(nw), b2 = f2_unpack(wr);
                            const float ya = __shfl_sync(0xffffffffu, a2.y, (lane - 1) & 31);
                            const float yb = __shfl_sync(0xffffffffu, b2.y, (lane - 1) & 31);
                            // lane 0: lane 31's wrapped second halves lie on diagonal C (its own)
                            emit_pos(C + lane, a2.x + (lane == 0 ? yb : ya));
                            emit_pos(C + lane - 32, b2.x + (lane == 0 ? 0.f : yb));
                        }
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&bars->ds_free[sb]);
                if (warp == 12) TRACE_FB(6, sc);
            }
        }
        if (lane == 0) bulk_wait0();
        __syncwarp();
        if (a.dpos) {   // the far entry: one atomic per warp
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) far_acc += __shfl_xor_sync(0xffffffffu, far_acc, off);
            if (lane == 0 && far_acc != 0.f) atomicAdd(a.dpos + a.P - 1, far_acc * rscale);
        }
    }
    __syncthreads();
    if (warp == 2) tmem_dealloc<512>(tmem);
}

// dQ = alpha/(2N) * acc (x gate), bf16, into its slice of dH
__global__ void __launch_bounds__(256) dq_finish_k(int64_t T, int width, const float* __restrict__ acc, int64_t lda,
                                                   const __nv_bfloat16* __restrict__ gate, int64_t ldg, float scale,
                                                   __nv_bfloat16* __restrict__ dq, int64_t ldq) {
    const int nch = width / 8;
    const int64_t total = T * nch;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = i / nch;
        const int c = (int)(i - row * nch) * 8;
        const float4 a0 = __ldcs(reinterpret_cast<const float4*>(acc + row * lda + c));
        const float4 a1 = __ldcs(reinterpret_cast<const float4*>(acc + row * lda + c + 4));
        float v[8] = {a0.x * scale, a0.y * scale, a0.z * scale, a0.w * scale,
                      a1.x * scale, a1.y * scale, a1.z * scale, a1.w * scale};
        if (gate) {
            const uint4 g = __ldg(reinterpret_cast<const uint4*>(gate + row * ldg + c));
            const __nv_bfloat162* g2 = reinterpret_cast<const __nv_bfloat162*>(&g);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const float2 f = __bfloat1622float2(g2[e]);
                v[2 * e] *= f.x;
                v[2 * e + 1] *= f.y;
            }
        }
        *reinterpret_cast<uint4*>(dq + row * ldq + c) =
            make_uint4(pack_bf16(v[0], v[1]), pack_bf16(v[2], v[3]), pack_bf16(v[4], v[5]), pack_bf16(v[6], v[7]));
    }
}
}  // namespace fb


}  // namespace

uh_status attn_bwd_sm100_launch(const AttnArgs& akv, cudaStream_t st, int64_t T) {
    if (akv.dh != DH) return fail(UH_ERR_UNSUPPORTED, "bf16 attention requires head_dim == 128");
    if (akv.n_items == 0) return UH_OK;
    const uint64_t width = (uint64_t)akv.H * DH;
    const int sms = num_sms();
    CUtensorMap q64, dA64, k128, v128, dqm;
    UH_TRY(make_tmap_bf16(&q64, akv.q, width, T, akv.ld_qkv, 64, fb::BN));
    UH_TRY(make_tmap_bf16(&dA64, akv.dout, width, T, akv.ld_dout, 64, fb::BN));
    UH_TRY(make_tmap_bf16(&k128, akv.k, width, T, akv.ld_qkv, 64, 128));
    UH_TRY(make_tmap_bf16(&v128, akv.v, width, T, akv.ld_qkv, 64, 128));
    UH_TRY(make_tmap_f32(&dqm, akv.dq_acc, width, T, akv.ld_acc, 32, 32));
    UH_CUDA(cudaMemsetAsync(akv.dq_acc, 0, (size_t)T * akv.ld_acc * sizeof(float), st));
    UH_CUDA(cudaFuncSetAttribute(fb::attn_bwd_fused_sm100, cudaFuncAttributeMaxDynamicSharedMemorySize, fb::SMEM));
    fb::attn_bwd_fused_sm100<<<akv.n_items < sms ? akv.n_items : sms, fb::THREADS, fb::SMEM, st>>>(
        q64, k128, v128, dA64, dqm, akv);
    note_launch();
    UH_CUDA(cudaGetLastError());
    fb::dq_finish_k<<<4 * sms, 256, 0, st>>>(T, (int)width, akv.dq_acc, akv.ld_acc,
                                             (const __nv_bfloat16*)akv.gq, akv.ld_gate, 0.5f * akv.alpha * akv.inv_n,
                                             (__nv_bfloat16*)akv.dq, akv.ld_grad);
    note_launch();
    UH_CUDA(cudaGetLastError());
    return UH_OK;
}

}  // namespace uh

#if UH_TRACE
extern "C" __attribute__((visibility("default"))) int uh_trace_set_bwd(long long* p) {
    return (int)cudaMemcpyToSymbol(uh::g_trace, &p, sizeof(p));
}
#endif
