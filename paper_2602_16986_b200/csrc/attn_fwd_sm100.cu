// attn_fwd_sm100.cu — fused jagged semi-local HSTU attention forward on tcgen05.
//
//   S = alpha * Q K^T + rab ;  P = silu(S) masked (select, never -inf) ;  A = (P V) / N
//   (Eq. 3; SLA mask P:140-146; pointwise SiLU, no softmax, P:85/P:90;
//    1/N and rab are readings R5/R7 of DESIGN.md; 1/N is applied once to the fp32
//    accumulator instead of to every score)
//
// One work item = (sequence, head, 128-query tile).  Only the 64-key tiles the SLA
// mask can reach are visited (global tiles, then the band; de-duplicated), so the
// work is O((K1 + K2) L) as the paper states.  No online-softmax state:
// O accumulates in TMEM across all visited tiles with no rescale.
//
// Warp roles (512 threads, one CTA per SM, persistent over the LPT-ordered items):
//   warp 0       TMA producer: Q tile once per item, (K,V) 64-key tiles through a 6-stage ring
//   warp 1       MMA issuer:   Q smem -> TMEM once per item (tcgen05.cp); S[b] = Q K^T (TS: Q in
//                TMEM, K from smem, N = 64); O += P V (TS: P over the consumed S columns, V MN-major)
//   warp 2       TMEM allocator (512 columns: S0..S4 at 0/64/.../256, O at 320, Q at 448)
//   warps 4-19   epilogue: four warpgroups, tile j to warpgroup j % 4 (S buffer j % 5);
//                per 32-column chunk TMEM -> regs -> (alpha, rab, mask: warp-uniform fast
//                path per chunk) -> silu via one tanh.approx -> bf16 P back into TMEM
//                (tcgen05.st); at the end of an item each warpgroup moves 32 O columns
//                TMEM -> x 1/N -> bf16 A rows.
// S has five TMEM buffers: the MMA issues S(j) four tiles ahead of PV(j), so four tiles'
// epilogues are in flight at once (one per warpgroup) and each warpgroup's next S is already
// issued while it finishes its current tile (five buffers over four warpgroups: cfg3 1.079 ->
// 1.035 ms; full causal without rab 1.10 -> 1.22 ms, the longer S-to-PV lag holding K/V stages).  The epilogue is latency-bound (a
// warpgroup puts one warp on each sub-partition): cfg3 forward 1.284 ms with two
// warpgroups, 1.173 with three, 1.111 with four (full causal with rab 1.601 -> 1.379 from
// three to four; without rab four are 2-7% slower than three).
#include <climits>

#include "attn_common.cuh"
#include "internal.h"

namespace uh {
namespace {

constexpr int BM = 128, BN = 64, DH = 128;
constexpr int QT = BM * DH * 2;          // 32 KB: Q tile, two 64-column swizzled blocks of 16 KB
constexpr int KT = BN * DH * 2;          // 16 KB: K (or V) tile, two 8 KB blocks
constexpr int PT = BM * BN * 2;          // 16 KB: P tile, one block
// (K,V) smem ring: the K of tile j loads once PV(j - STAGES) has completed; with four
// epilogue warpgroups 5 -> 6 stages is cfg3-neutral and takes full causal from 1.23 to 1.07 ms
constexpr int STAGES = 6;
constexpr int NS = 5;                   // S buffers in TMEM (64 columns each)
constexpr int LAG = NS - 1;             // the MMA issues S(j) LAG tiles ahead of PV(j)
constexpr int O_COL = 320;              // TMEM column of the O accumulator
constexpr int Q_COL = 448;              // TMEM columns of Q (A operand of S = Q K^T), 64 packed columns
constexpr int NUM_THREADS = 640;
// registers per thread after setmaxnreg (640 threads start at 96): the control warpgroup gives
// up 32, the four epilogue warpgroups take 8 more (an increase is served only from the CTA's
// own releases: 128 x (96 - 64) >= 512 x (104 - 96))
constexpr int REG_CTRL = 64, REG_EPI = 104;
static_assert(128 * (96 - REG_CTRL) >= 512 * (REG_EPI - 96), "setmaxnreg: the epilogue increase must fit");
constexpr int SMEM_BYTES = QT + STAGES * 2 * KT + 256 + 1024 + 512;

struct __align__(8) FwdBars {
    uint64_t q_full, q_empty;
    uint64_t kv_full[STAGES], kv_empty[STAGES];
    uint64_t s_full[NS];
    uint64_t p_full[NS];
    uint64_t o_full, o_empty;
    ItemRing ring;
    uint32_t tmem;
};

__device__ __forceinline__ void store_bf16_row32(uint8_t* tile, int r, int col0, const float* v) {
    uint8_t* row = tile + r * 128;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        const int ch = (col0 >> 3) + c;
        uint4 u = make_uint4(pack_bf16(v[c * 8 + 0], v[c * 8 + 1]), pack_bf16(v[c * 8 + 2], v[c * 8 + 3]),
                             pack_bf16(v[c * 8 + 4], v[c * 8 + 5]), pack_bf16(v[c * 8 + 6], v[c * 8 + 7]));
        *reinterpret_cast<uint4*>(row + ((ch ^ (r & 7)) << 4)) = u;
    }
}

__global__ void __launch_bounds__(NUM_THREADS, 1)
attn_fwd_sm100(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
               const __grid_constant__ CUtensorMap tmV, AttnArgs a) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sQ = smem;
    uint8_t* sKV = smem + QT;                     // [STAGES] x (K 16K | V 16K)
    float* ts_s = reinterpret_cast<float*>(sKV + STAGES * 2 * KT);   // time_bias / 2 [32]
    FwdBars* bars = reinterpret_cast<FwdBars*>(ts_s + 64);

    const int warp = threadIdx.x >> 5;
    TRACE_SETUP();
    const int lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        mbar_init(&bars->q_full, 1); mbar_init(&bars->q_empty, 1);
        for (int i = 0; i < STAGES; ++i) { mbar_init(&bars->kv_full[i], 1); mbar_init(&bars->kv_empty[i], 1); }
        for (int i = 0; i < NS; ++i) { mbar_init(&bars->s_full[i], 1); mbar_init(&bars->p_full[i], 4); }
        mbar_init(&bars->o_full, 1); mbar_init(&bars->o_empty, 16);
        ring_init(&bars->ring, 17);   // MMA warp + 16 epilogue warps
        fence_barrier_init();
    }
    stage_ts(a, ts_s);
    if (warp == 0 && lane == 0) { tma_prefetch_desc(&tmQ); tma_prefetch_desc(&tmK); tma_prefetch_desc(&tmV); }
    if (warp == 2) tmem_alloc<512>(&bars->tmem);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = bars->tmem;

    if (warp < 4) {
    // control warpgroup: TMA producer (warp 0), MMA issuer (warp 1), TMEM allocator (warp 2)
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(REG_CTRL));
    if (warp == 0) {
        // ============================================================ producer
        if (lane == 0) {
            int kc = 0, qi = 0;
            for (;; ++qi) {
                const int w = ring_claim_publish(&bars->ring, qi, a.counter, a.n_items);
                if (w < 0) break;
                const WorkItem it = a.items[w];
                check_item(a, it, BM);
                const int q0 = it.tile * BM, h = it.head & 0xFFFF;
                const KeyTiles kt = key_tiles(q0, BM, it.seq_len, a.K1, a.K2, BN);
                const int n = key_tiles_count(kt);
                mbar_wait_sleep(&bars->q_empty, (qi & 1) ^ 1);
                mbar_arrive_expect_tx(&bars->q_full, QT);
                tma_load_2d(sQ, &tmQ, &bars->q_full, h * DH, it.seq_start + q0);
                tma_load_2d(sQ + QT / 2, &tmQ, &bars->q_full, h * DH + 64, it.seq_start + q0);
                for (int j = 0; j < n; ++j) {
                    const int row = it.seq_start + key_tile_at(kt, j) * BN;
                    const int s = kc % STAGES;
                    uint8_t* st = sKV + s * 2 * KT;
                    mbar_wait_sleep(&bars->kv_empty[s], ((kc / STAGES) & 1) ^ 1);
                    TRACE(7 * 1024 + (kc & 1023));   // stage free: PV(kc - STAGES) done
                    mbar_arrive_expect_tx(&bars->kv_full[s], 2 * KT);
                    tma_load_2d(st, &tmK, &bars->kv_full[s], h * DH, row);
                    tma_load_2d(st + KT / 2, &tmK, &bars->kv_full[s], h * DH + 64, row);
                    tma_load_2d(st + KT, &tmV, &bars->kv_full[s], h * DH, row);
                    tma_load_2d(st + KT + KT / 2, &tmV, &bars->kv_full[s], h * DH + 64, row);
                    ++kc;
                }
            }
        }
    } else if (warp == 1) {
        // ============================================================ MMA issuer
        constexpr uint32_t idesc_s = make_idesc_bf16(BM, BN, false, false);  // Q (K-major) x K (K-major)
        constexpr uint32_t idesc_o = make_idesc_bf16(BM, DH, false, true);   // P (K-major) x V (MN-major)
        int kc = 0, sc = 0, pc = 0, qi = 0;
        const uint32_t q_addr = smem_u32(sQ);
        for (;; ++qi) {
            const int w = ring_take(&bars->ring, qi, lane);
            if (w < 0) break;
            const WorkItem it = a.items[w];
            check_item(a, it, BM);
            const KeyTiles kt = key_tiles(it.tile * BM, BM, it.seq_len, a.K1, a.K2, BN);
            const int n = key_tiles_count(kt);
            const int kc0 = kc;
            mbar_wait(&bars->q_full, qi & 1);
            tc_fence_after();
            if (elect_one()) {   // Q: smem -> TMEM once per item (in order with the MMAs that read it)
#pragma unroll
                for (int kk = 0; kk < DH / 16; ++kk)
                    tmem_cp_128x256b(tmem + Q_COL + kk * 8,
                                     make_sw128_desc(q_addr + (kk >> 2) * (QT / 2) + (kk & 3) * 32, 16, 1024));
                umma_commit(&bars->q_empty);
            }
            __syncwarp();
            // S(j) runs LAG tiles ahead of PV(j - LAG).  The barrier of the next block is probed
            // (mbarrier.test_wait, never parks) just before the current block's MMAs are issued and
            // only then waited on, so an already-complete barrier costs no pipe idle time.
            // Incremental ring state: S side (kv stage / phase, S buffer), PV side (kv stage,
            // P buffer / phase).
            int s_st = kc % STAGES, s_ph = (kc / STAGES) & 1, s_sb = sc % NS;
            int p_st = s_st, p_b = pc % NS, p_ph = (pc / NS) & 1;
            mbar_wait(&bars->kv_full[s_st], s_ph);
            for (int j = 0; j < n + LAG; ++j) {
                if (j < n) {   // ---- S(j) = Q K_j^T  (buffer s_sb last read by PV(j - NS): the pipe is in order)
                    tc_fence_after();
                    // next block: PV(j - LAG) if it exists, else S(j + 1), else PV(0) (n <= LAG)
                    const bool nxt_p = j >= LAG || j + 1 >= n;
                    const int ns_st = s_st + 1 == STAGES ? 0 : s_st + 1, ns_ph = s_st + 1 == STAGES ? s_ph ^ 1 : s_ph;
                    uint64_t* nb = nxt_p ? &bars->p_full[p_b] : &bars->kv_full[ns_st];
                    const uint32_t np = nxt_p ? p_ph : ns_ph;
                    const bool rdy = mbar_test(smem_u32(nb), np);
                    if (lane == 0) TRACE(0 * 1024 + ((kc0 + j) & 1023));
                    if (elect_one()) {
                        const uint32_t k_addr = smem_u32(sKV + s_st * 2 * KT);
#pragma unroll
                        for (int kk = 0; kk < DH / 16; ++kk)
                            umma_ts(tmem + s_sb * BN, tmem + Q_COL + kk * 8,
                                    make_sw128_desc(k_addr + (kk >> 2) * (KT / 2) + (kk & 3) * 32, 16, 1024), idesc_s,
                                    kk > 0 ? 1u : 0u);
                        umma_commit(&bars->s_full[s_sb]);
                    }
                    __syncwarp();
                    s_st = ns_st; s_ph = ns_ph;
                    s_sb = s_sb + 1 == NS ? 0 : s_sb + 1;
                    if (!rdy) mbar_wait(nb, np);
                }
                if (j >= LAG) {   // ---- O += P(jj) V_jj  (P over the consumed S columns: keys [32g, 32g+32) at col 32g)
                    const int jj = j - LAG;
                    if (jj == 0) mbar_wait(&bars->o_empty, (qi & 1) ^ 1);
                    tc_fence_after();
                    // next block: S(j + 1) if it exists, else PV(jj + 1) if it exists, else none
                    const bool nxt_s = j + 1 < n;
                    const int np_b = p_b + 1 == NS ? 0 : p_b + 1, np_ph = p_b + 1 == NS ? p_ph ^ 1 : p_ph;
                    uint64_t* nb = nxt_s ? &bars->kv_full[s_st] : &bars->p_full[jj + 1 < n ? np_b : p_b];
                    const uint32_t np = nxt_s ? s_ph : (jj + 1 < n ? np_ph : p_ph);
                    const bool rdy = mbar_test(smem_u32(nb), np);
                    if (lane == 0) TRACE(1 * 1024 + ((kc0 + jj) & 1023));
                    if (elect_one()) {
                        const uint32_t v_addr = smem_u32(sKV + p_st * 2 * KT + KT);
#pragma unroll
                        for (int kk = 0; kk < BN / 16; ++kk)
                            umma_ts(tmem + O_COL, tmem + p_b * BN + (kk >> 1) * 32 + (kk & 1) * 8,
                                    make_sw128_desc(v_addr + kk * 2048, KT / 2, 1024), idesc_o,
                                    (jj > 0 || kk > 0) ? 1u : 0u);
                        umma_commit(&bars->kv_empty[p_st]);
                        if (jj == n - 1) umma_commit(&bars->o_full);
                    }
                    __syncwarp();
                    p_st = p_st + 1 == STAGES ? 0 : p_st + 1;
                    p_b = np_b; p_ph = np_ph;
                    if (!rdy) mbar_wait(nb, np);
                }
            }
            kc += n; sc += n; pc += n;
        }
    }
    } else {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(REG_EPI));
        // ============================================================ epilogue
        const int wg = (warp - 4) >> 2;      // warpgroup: handles the tiles j with j % 4 == wg
        const int wq = warp & 3;             // TMEM lane quarter
        const int r = wq * 32 + lane;        // row of the tile
        const uint32_t lane_base = (uint32_t)(wq * 32) << 16;
        const float ha = 0.5f * a.alpha;
        int sc = 0, qi = 0;
        int w = ring_take(&bars->ring, 0, lane);
        WorkItem itn{};
        int64_t t0n = 0, tqn = 0;    // the next item's first timestamp and this row's (raw)
        auto load_rowtimes = [&](const WorkItem& x) {
            if (a.ts) {
                t0n = __ldg(a.t + x.seq_start);
                tqn = __ldg(a.t + x.seq_start + imin(x.tile * BM + r, x.seq_len - 1));
            }
        };
        if (w >= 0) { itn = a.items[w]; load_rowtimes(itn); }
        const float pos_far = a.pos ? 0.5f * __ldg(a.pos + a.P - 1) : 0.f;
        for (;; ++qi) {
            if (w < 0) break;
            const WorkItem it = itn;
            check_item(a, it, BM);
            const int L = it.seq_len, o = it.seq_start, h = it.head & 0xFFFF;
            const int q0 = it.tile * BM;
            const KeyTiles kt = key_tiles(q0, BM, L, a.K1, a.K2, BN);
            const int n = key_tiles_count(kt);
            const int qp = q0 + r;
            const bool qok = qp < L;
            ChunkCtx cx;
            cx.pe = a.pos ? a.pos_ext + kPosOff : nullptr;
            cx.Lt = a.pos_ext_len;
            cx.pos_far = pos_far;
            cx.P = a.P;
            cx.ts_h = a.ts ? ts_s : nullptr;
            cx.NB = a.NB;
            cx.t = a.t ? a.t + o : nullptr;
            cx.t0 = a.ts ? t0n : 0;
            cx.K1 = a.K1; cx.K2 = a.K2; cx.L = L;
            cx.ha = 0.5f * a.alpha;
            const int32_t tq = (a.ts && qok) ? rel32(tqn, cx.t0) : 0;
            // tiles rotate over the four warpgroups (global tile index mod 4), so one group's
            // SiLU burst overlaps the others' TMEM traffic, loads and bookkeeping
            for (int j = 0; j < n; ++j, ++sc) {
                if ((sc & 3) != wg) continue;
                const int sb = sc % NS;
                const int k0 = key_tile_at(kt, j) * BN;
                const int32_t tc0 = col_time(cx, k0, lane), tc1 = col_time(cx, k0 + 32, lane);
                if (warp == 4 && lane == 0) TRACE(2 * 1024 + (sc & 1023));
                mbar_wait_sleep(&bars->s_full[sb], (sc / NS) & 1);
                if (warp == 4 && lane == 0) TRACE(3 * 1024 + (sc & 1023));
                if (warp == 8 && lane == 0) TRACE(6 * 1024 + (sc & 1023));
                tc_fence_after();
#pragma unroll
                for (int hc = 0; hc < 2; ++hc) {
                    const int kb = k0 + 32 * hc;
                    const Chunk ch = q_chunk(cx, qp, qok, tq, kb, hc ? tc1 : tc0);
                    float s[32];
                    tmem_ld32(tmem + lane_base + sb * BN + 32 * hc, s);
                    tmem_ld_wait();
                    // h = (alpha S + rab)/2 in fp32, then packed bf16x2: silu(2h) = h + h tanh(h)
                    float hx[32];
                    q_h(cx, ch, tq, s, hx);
                    if (ch.flags & FLAG_M) apply_vis(hx, q_vis_bits(cx, qp, qok, kb));   // h = 0 -> P = 0
                    uint32_t pk[16];
#pragma unroll
                    for (int i = 0; i < 16; ++i) {   // fp32 tanh, h + h t as one packed FFMA2, one bf16 pack
                        const uint64_t H = f2_pack(hx[2 * i], hx[2 * i + 1]);
                        const float2 p2 = f2_unpack(ffma2(H, f2_pack(tanh_approx(hx[2 * i]), tanh_approx(hx[2 * i + 1])), H));
                        pk[i] = pack_bf16(p2.x, p2.y);
                    }
                    // P -> TMEM over the chunk's own (already read) S columns: keys [32hc, 32hc+32) at col 32hc
                    tmem_st16(tmem + lane_base + sb * BN + 32 * hc, pk);
                }
                if (warp == 4 && lane == 0) TRACE(4 * 1024 + (sc & 1023));
                tmem_st_wait();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&bars->p_full[sb]);
                if (warp == 4 && lane == 0) TRACE(5 * 1024 + (sc & 1023));
            }
            // the next item before this one's O epilogue (the o_full wait hides its loads)
            const int wn = ring_take(&bars->ring, qi + 1, lane);
            if (wn >= 0) {
                itn = a.items[wn];
                load_rowtimes(itn);
                if (a.ts) {
                    const int on = itn.seq_start, qn = itn.tile * BM;
                    const KeyTiles ktn = key_tiles(qn, BM, itn.seq_len, a.K1, a.K2, BN);
                    const int j0 = (wg - sc) & 3;   // this warpgroup's first tile of the next item
                    const int64_t* tp = a.t + on;
                    asm volatile("prefetch.global.L1 [%0];" ::"l"(tp));
                    asm volatile("prefetch.global.L1 [%0];" ::"l"(tp + imin(qn + r, itn.seq_len - 1)));
                    if (j0 < key_tiles_count(ktn)) {
                        const int kb = key_tile_at(ktn, j0) * BN;
                        asm volatile("prefetch.global.L1 [%0];" ::"l"(tp + imin(kb + lane, itn.seq_len - 1)));
                        asm volatile("prefetch.global.L1 [%0];" ::"l"(tp + imin(kb + 32 + lane, itn.seq_len - 1)));
                    }
                }
            }
            w = wn;
            // ---- O epilogue: A = O / N (32 columns per warpgroup)
            mbar_wait_sleep(&bars->o_full, qi & 1);
            tc_fence_after();
            float ov[32];
            tmem_ld32(tmem + lane_base + O_COL + wg * 32, ov);
            tmem_ld_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&bars->o_empty);
            UH_CHECK(!qok || (int64_t)o + qp < a.T);
            const bool v8 = ((reinterpret_cast<uintptr_t>(a.out) | (uintptr_t)(a.ld_out * 2)) & 31) == 0;
            if (qok && v8) {
                uint32_t* op = reinterpret_cast<uint32_t*>(reinterpret_cast<__nv_bfloat16*>(a.out) +
                                                           (int64_t)(o + qp) * a.ld_out + h * DH + wg * 32);
                const float sN = a.inv_n;
#pragma unroll
                for (int hv = 0; hv < 2; ++hv) {
                    uint32_t w8[8];
#pragma unroll
                    for (int e = 0; e < 8; ++e)
                        w8[e] = pack_bf16(ov[hv * 16 + 2 * e] * sN, ov[hv * 16 + 2 * e + 1] * sN);
                    asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(op + hv * 8),
                                 "r"(w8[0]), "r"(w8[1]), "r"(w8[2]), "r"(w8[3]), "r"(w8[4]), "r"(w8[5]), "r"(w8[6]),
                                 "r"(w8[7]) : "memory");
                }
            } else if (qok) {
                uint4* op = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(a.out) +
                                                     (int64_t)(o + qp) * a.ld_out + h * DH + wg * 32);
                const float sN = a.inv_n;
#pragma unroll
                for (int ch = 0; ch < 4; ++ch)
                    op[ch] = make_uint4(pack_bf16(ov[ch * 8 + 0] * sN, ov[ch * 8 + 1] * sN),
                                        pack_bf16(ov[ch * 8 + 2] * sN, ov[ch * 8 + 3] * sN),
                                        pack_bf16(ov[ch * 8 + 4] * sN, ov[ch * 8 + 5] * sN),
                                        pack_bf16(ov[ch * 8 + 6] * sN, ov[ch * 8 + 7] * sN));
            }
        }
    }
    __syncthreads();
    if (warp == 2) tmem_dealloc<512>(tmem);
}

}  // namespace

uh_status attn_fwd_sm100_launch(const AttnArgs& a, cudaStream_t st, int64_t T) {
    if (a.n_items == 0) return UH_OK;
    if (a.dh != DH) return fail(UH_ERR_UNSUPPORTED, "bf16 attention requires head_dim == 128");
    const uint64_t width = (uint64_t)a.H * DH;
    CUtensorMap tq, tk, tv;
    UH_TRY(make_tmap_bf16(&tq, a.q, width, (uint64_t)T, a.ld_qkv, 64, BM));
    UH_TRY(make_tmap_bf16(&tk, a.k, width, (uint64_t)T, a.ld_qkv, 64, BN));
    UH_TRY(make_tmap_bf16(&tv, a.v, width, (uint64_t)T, a.ld_qkv, 64, BN));
    UH_CUDA(cudaFuncSetAttribute(attn_fwd_sm100, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES));
    const int grid = a.n_items < num_sms() ? a.n_items : num_sms();
    attn_fwd_sm100<<<grid, NUM_THREADS, SMEM_BYTES, st>>>(tq, tk, tv, a);
    note_launch();
    UH_CUDA(cudaGetLastError());
    return UH_OK;
}

}  // namespace uh

#if UH_TRACE
extern "C" __attribute__((visibility("default"))) int uh_trace_set(long long* p) {
    return (int)cudaMemcpyToSymbol(uh::g_trace, &p, sizeof(p));
}
#endif
