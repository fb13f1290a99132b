// attn_fwd_sm100.cu — fused jagged semi-local HSTU attention forward on tcgen05.
//
//   S = alpha * Q K^T + rab ;  P = (silu(S) / N) masked (select, never -inf) ;  O = P V
//   (Eq. 3; SLA mask P:140-146; pointwise SiLU, no softmax, P:85/P:90;
//    1/N and rab are readings R5/R7 of DESIGN.md)
//
// One work item = (sequence, head, 128-query tile).  Only the key tiles the SLA
// mask can reach are visited (global tiles, then the band; de-duplicated), so the
// work is O((K1 + K2) L) as the paper states.  No online-softmax state:
// O accumulates in TMEM across all visited tiles with no rescale.
//
// Warp roles (384 threads):
//   warp 0       TMA producer: Q tile once per item, K/V tiles through 2-stage rings
//   warp 1       MMA issuer:   S[b] = Q K^T (SS, K-major), O += P V (P K-major, V MN-major)
//   warp 2       TMEM allocator (512 columns: S0 | S1 | O | spare)
//   warps 4-11   epilogue: two warpgroups, each owns 64 of the 128 key columns of S:
//                TMEM -> regs, scale + rab + mask + SiLU/N -> bf16 P (swizzled smem),
//                and at the end of an item O TMEM -> bf16 A rows.
// S is double-buffered in TMEM so the MMA of S_{j+1} overlaps the epilogue of S_j.
#include <climits>

#include "attn_common.cuh"
#include "internal.h"

namespace uh {
namespace {

constexpr int BM = 128, BN = 128, DH = 128;
constexpr int TILE_BYTES = 128 * 128 * 2;  // 32 KB: one 128x128 bf16 tile = 2 swizzled 64-col blocks
constexpr int HALF_BYTES = TILE_BYTES / 2;
constexpr int NUM_THREADS = 384;
constexpr int SMEM_BYTES = 7 * TILE_BYTES + 1024 + 512;

struct __align__(8) FwdBars {
    uint64_t q_full, q_empty;
    uint64_t k_full[2], k_empty[2];
    uint64_t v_full[2], v_empty[2];
    uint64_t s_full[2], s_empty[2];
    uint64_t p_full[2], p_empty[2];
    uint64_t o_full, o_empty;
    uint32_t tmem;
};

__device__ __forceinline__ void load_tile(uint8_t* dst, const CUtensorMap* m, uint64_t* bar, int col, int row) {
    tma_load_2d(dst, m, bar, col, row);
    tma_load_2d(dst + HALF_BYTES, m, bar, col + 64, row);
}

__global__ void __launch_bounds__(NUM_THREADS, 1)
attn_fwd_sm100(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
               const __grid_constant__ CUtensorMap tmV, AttnArgs a) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sQ = smem;
    uint8_t* sK = smem + TILE_BYTES;        // [2]
    uint8_t* sV = smem + 3 * TILE_BYTES;    // [2]
    uint8_t* sP = smem + 5 * TILE_BYTES;    // [2]
    FwdBars* bars = reinterpret_cast<FwdBars*>(smem + 7 * TILE_BYTES);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        mbar_init(&bars->q_full, 1); mbar_init(&bars->q_empty, 1);
        for (int i = 0; i < 2; ++i) {
            mbar_init(&bars->k_full[i], 1); mbar_init(&bars->k_empty[i], 1);
            mbar_init(&bars->v_full[i], 1); mbar_init(&bars->v_empty[i], 1);
            mbar_init(&bars->s_full[i], 1); mbar_init(&bars->s_empty[i], 8);
            mbar_init(&bars->p_full[i], 8); mbar_init(&bars->p_empty[i], 1);
        }
        mbar_init(&bars->o_full, 1); mbar_init(&bars->o_empty, 8);
        fence_barrier_init();
    }
    if (warp == 0 && lane == 0) { tma_prefetch_desc(&tmQ); tma_prefetch_desc(&tmK); tma_prefetch_desc(&tmV); }
    if (warp == 2) tmem_alloc<512>(&bars->tmem);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = bars->tmem;

    if (warp == 0) {
        // ============================================================ producer
        if (lane == 0) {
            int kc = 0, vc = 0, qi = 0;
            for (int w = blockIdx.x; w < a.n_items; w += gridDim.x, ++qi) {
                const WorkItem it = a.items[w];
                const int q0 = it.tile * BM, h = it.head & 0xFFFF;
                const KeyTiles kt = key_tiles(q0, BM, it.seq_len, a.K1, a.K2, BN);
                const int n = key_tiles_count(kt);
                mbar_wait(&bars->q_empty, (qi & 1) ^ 1);
                mbar_arrive_expect_tx(&bars->q_full, TILE_BYTES);
                load_tile(sQ, &tmQ, &bars->q_full, h * DH, it.seq_start + q0);
                for (int j = 0; j < n; ++j) {
                    const int row = it.seq_start + key_tile_at(kt, j) * BN;
                    const int ks = kc & 1;
                    mbar_wait(&bars->k_empty[ks], ((kc >> 1) & 1) ^ 1);
                    mbar_arrive_expect_tx(&bars->k_full[ks], TILE_BYTES);
                    load_tile(sK + ks * TILE_BYTES, &tmK, &bars->k_full[ks], h * DH, row);
                    ++kc;
                    const int vs = vc & 1;
                    mbar_wait(&bars->v_empty[vs], ((vc >> 1) & 1) ^ 1);
                    mbar_arrive_expect_tx(&bars->v_full[vs], TILE_BYTES);
                    load_tile(sV + vs * TILE_BYTES, &tmV, &bars->v_full[vs], h * DH, row);
                    ++vc;
                }
            }
        }
    } else if (warp == 1) {
        // ============================================================ MMA issuer
        constexpr uint32_t idesc_s = make_idesc_bf16(BM, BN, false, false);  // Q (K-major) x K (K-major)
        constexpr uint32_t idesc_o = make_idesc_bf16(BM, DH, false, true);   // P (K-major) x V (MN-major)
        int kc = 0, vc = 0, sc = 0, pc = 0, qi = 0;
        const uint32_t q_addr = smem_u32(sQ);
        auto issue_pv = [&](int jj) {
            const int pb = pc & 1, vs = vc & 1;
            mbar_wait(&bars->p_full[pb], (pc >> 1) & 1);
            mbar_wait(&bars->v_full[vs], (vc >> 1) & 1);
            tc_fence_after();
            if (elect_one()) {
                const uint32_t p_addr = smem_u32(sP + pb * TILE_BYTES);
                const uint32_t v_addr = smem_u32(sV + vs * TILE_BYTES);
#pragma unroll
                for (int kk = 0; kk < BN / 16; ++kk) {
                    uint64_t ad = make_sw128_desc(p_addr + (kk >> 2) * HALF_BYTES + (kk & 3) * 32, 16, 1024);
                    uint64_t bd = make_sw128_desc(v_addr + kk * 2048, HALF_BYTES, 1024);
                    umma_ss(tmem + 256, ad, bd, idesc_o, (jj > 0 || kk > 0) ? 1u : 0u);
                }
                umma_commit(&bars->p_empty[pb]);
                umma_commit(&bars->v_empty[vs]);
            }
            __syncwarp();
            ++pc; ++vc;
        };
        for (int w = blockIdx.x; w < a.n_items; w += gridDim.x, ++qi) {
            const WorkItem it = a.items[w];
            const KeyTiles kt = key_tiles(it.tile * BM, BM, it.seq_len, a.K1, a.K2, BN);
            const int n = key_tiles_count(kt);
            mbar_wait(&bars->q_full, qi & 1);
            for (int j = 0; j < n; ++j) {
                const int ks = kc & 1, sb = sc & 1;
                mbar_wait(&bars->k_full[ks], (kc >> 1) & 1);
                mbar_wait(&bars->s_empty[sb], ((sc >> 1) & 1) ^ 1);
                tc_fence_after();
                if (elect_one()) {
                    const uint32_t k_addr = smem_u32(sK + ks * TILE_BYTES);
#pragma unroll
                    for (int kk = 0; kk < DH / 16; ++kk) {
                        const uint32_t off = (kk >> 2) * HALF_BYTES + (kk & 3) * 32;
                        umma_ss(tmem + sb * BN, make_sw128_desc(q_addr + off, 16, 1024),
                                make_sw128_desc(k_addr + off, 16, 1024), idesc_s, kk > 0 ? 1u : 0u);
                    }
                    umma_commit(&bars->k_empty[ks]);
                    umma_commit(&bars->s_full[sb]);
                    if (j == n - 1) umma_commit(&bars->q_empty);
                }
                __syncwarp();
                ++kc; ++sc;
                if (j >= 1) {
                    if (j == 1) { mbar_wait(&bars->o_empty, (qi & 1) ^ 1); }
                    issue_pv(j - 1);
                }
            }
            if (n == 1) mbar_wait(&bars->o_empty, (qi & 1) ^ 1);
            issue_pv(n - 1);
            if (elect_one()) umma_commit(&bars->o_full);
            __syncwarp();
        }
    } else if (warp >= 4) {
        // ============================================================ epilogue
        const int wg = (warp - 4) >> 2;      // column half: keys [64*wg, 64*wg+64) of the tile
        const int wq = warp & 3;             // TMEM lane quarter
        const int r = wq * 32 + lane;        // row of the tile
        const uint32_t lane_base = (uint32_t)(wq * 32) << 16;
        const float half_inv_n = 0.5f * a.inv_n;
        int sc = 0, pc = 0, qi = 0;
        for (int w = blockIdx.x; w < a.n_items; w += gridDim.x, ++qi) {
            const WorkItem it = a.items[w];
            const int L = it.seq_len, o = it.seq_start, h = it.head & 0xFFFF;
            const int q0 = it.tile * BM;
            const KeyTiles kt = key_tiles(q0, BM, L, a.K1, a.K2, BN);
            const int n = key_tiles_count(kt);
            const int qp = q0 + r;
            const bool qok = qp < L;
            const int64_t tq = (a.ts && qok) ? __ldg(a.t + o + qp) : 0;
            for (int j = 0; j < n; ++j) {
                const int kbase = key_tile_at(kt, j) * BN + wg * 64;
                const int sb = sc & 1;
                mbar_wait(&bars->s_full[sb], (sc >> 1) & 1);
                tc_fence_after();
                float s[64];
                tmem_ld32(tmem + lane_base + sb * BN + wg * 64, s);
                tmem_ld32(tmem + lane_base + sb * BN + wg * 64 + 32, s + 32);
                tmem_ld_wait();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&bars->s_empty[sb]);
                ++sc;
                // scale, bias, mask, SiLU / N
                const bool full_tile = qok && (kbase + 63 <= qp - 0) && (kbase + 63 < L) &&
                                       (qp - kbase <= a.K1 || kbase + 63 < a.K2);
#pragma unroll
                for (int c = 0; c < 64; ++c) {
                    const int kp = kbase + c;
                    float x = a.alpha * s[c];
                    bool ok = full_tile || (qok && kp < L && mask_ok(qp, kp, a.K1, a.K2));
                    if (a.pos || a.ts) {
                        int64_t tk = (a.ts && ok) ? __ldg(a.t + o + kp) : tq;
                        if (ok) x += rab_bias(a, qp, kp, tq, tk);
                    }
                    float hx = 0.5f * x;
                    float pv = x * half_inv_n * (1.0f + tanh_approx(hx));
                    s[c] = ok ? pv : 0.0f;
                }
                const int pb = pc & 1;
                mbar_wait(&bars->p_empty[pb], ((pc >> 1) & 1) ^ 1);
                uint8_t* prow = sP + pb * TILE_BYTES + wg * HALF_BYTES + r * 128;
#pragma unroll
                for (int ch = 0; ch < 8; ++ch) {
                    uint4 v = make_uint4(pack_bf16(s[ch * 8 + 0], s[ch * 8 + 1]), pack_bf16(s[ch * 8 + 2], s[ch * 8 + 3]),
                                         pack_bf16(s[ch * 8 + 4], s[ch * 8 + 5]), pack_bf16(s[ch * 8 + 6], s[ch * 8 + 7]));
                    *reinterpret_cast<uint4*>(prow + ((ch ^ (r & 7)) << 4)) = v;
                }
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) mbar_arrive(&bars->p_full[pb]);
                ++pc;
            }
            // ---- O epilogue
            mbar_wait(&bars->o_full, qi & 1);
            tc_fence_after();
            float ov[64];
            tmem_ld32(tmem + lane_base + 256 + wg * 64, ov);
            tmem_ld32(tmem + lane_base + 256 + wg * 64 + 32, ov + 32);
            tmem_ld_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&bars->o_empty);
            if (qok) {
                uint4* op = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(a.out) +
                                                     (int64_t)(o + qp) * a.ld_out + h * DH + wg * 64);
#pragma unroll
                for (int ch = 0; ch < 8; ++ch)
                    op[ch] = make_uint4(pack_bf16(ov[ch * 8 + 0], ov[ch * 8 + 1]), pack_bf16(ov[ch * 8 + 2], ov[ch * 8 + 3]),
                                        pack_bf16(ov[ch * 8 + 4], ov[ch * 8 + 5]), pack_bf16(ov[ch * 8 + 6], ov[ch * 8 + 7]));
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
