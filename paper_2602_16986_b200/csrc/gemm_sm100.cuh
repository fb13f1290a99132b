// gemm_sm100.cuh — persistent, warp-specialised tcgen05 GEMM for the layer's
// projections (f1, f2 and their backward products; Listing 1).
//
//   C[M,N] = A[M,K] * B[K,N]   (bf16 operands via TMA, fp32 accumulation in TMEM)
//
// A is "K-major" when stored [M][K] (row-major activations) and "MN-major" when
// stored [K][M] (the transposed operand of a weight gradient, e.g. x^T).  B is
// K-major when stored [N][K] and MN-major when stored [K][N].  Both majors map
// to the UMMA descriptor's major bits; no transpose copies are made.
//
// Epilogues (fused, so no standalone elementwise pass over [T,4d] exists):
//   EPI_BF16 : out0 = bf16(acc + bias[n] + resid[m,n])     f2 + 2-D residual
//   EPI_SILU : h = acc + bias[n]; out0 = bf16(silu(h)); out1 = bf16(silu'(h))  f1 + phi1 (Eq. 2)
//   EPI_F32  : atomically add acc into fp32 out0 (split-K weight gradients)
//
// Roles (384 threads): warp 0 TMA producer, warp 1 MMA issuer, warp 2 TMEM
// allocator, warps 4-11 epilogue in two warpgroups that split the BN columns
// (thread = TMEM lane = output row).  TMEM holds two
// BN-column accumulators so the epilogue of tile i overlaps the main loop of i+1.
#pragma once
#include "sm100.cuh"

namespace uh {

enum { EPI_BF16 = 0, EPI_SILU = 1, EPI_F32 = 2 };

struct GemmArgs {
    int M, N, K;
    int m_tiles, n_tiles, k_splits, kb_per_split;  // kb = 64-wide K blocks
    void* out0; int64_t ld0;
    void* out1; int64_t ld1;
    const float* bias;
    const __nv_bfloat16* resid; int64_t ldr;
    float* colsum;      // EPI_F32, 256-wide MN-major B: += column sums of B (the bias gradient), or null
    const float* scale_a = nullptr;   // F8: per-row scales of A [M]
    const float* scale_b = nullptr;   // F8: per-column scales of B [N]
};

// MSUB row sub-tiles of 128 share each B k-block (tile BM = 128 MSUB): for the long-K split-K
// weight gradients, a 256 x 256 tile streams 64 KB per 1024 MMA cycles instead of 128 x 128's
// 32 KB per 256 (L2->SM ingress is the limit there).  NACC TMEM accumulators (2 when they fit:
// the epilogue of tile i overlaps tile i+1's main loop).
// CG = 2: a CTA pair computes a 256 x BN tile with cta_group::2 MMAs (M = 256); each CTA holds
// its 128 A rows and BN/2 B columns per stage, so the per-SM operand traffic through shared
// memory is that of a 128 x BN/2 tile (the f1 GEMM's 128 x 256 tile is shared-memory bound).
template <int BN, int MSUB = 1, int EPI = 0, int CG = 1>
struct GemmCfg {
    static constexpr int BM = 128 * MSUB, BK = 64;
    static constexpr int STAGES = MSUB == 2 ? 3 : (BN / CG == 256 ? 4 : 6);
    static constexpr int A_BYTES = BM * BK * 2;
    static constexpr int B_BYTES = BN / CG * BK * 2;
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    // per epilogue warp a 32x32 bf16 box per output (TMA stores); EPI_F32: [8 row groups][BN] column-sum partials
    static constexpr int STAGING = EPI == 2 ? 8 * BN * 4 : 8 * 2 * 2048;
    static constexpr int SMEM = STAGES * STAGE_BYTES + STAGING + 1024 /*align*/ + 256 /*barriers*/;
    static constexpr int NACC = 2 * MSUB * BN <= 512 ? 2 : 1;
    static constexpr int TMEM_COLS = NACC * MSUB * BN <= 256 ? 256 : 512;
};

// F8 (NEXT-2): E4M3 A and B^T, both K-major, kind::f8f6f4; a K block is 128 elements (the same
// 128-byte rows, swizzle and descriptors as bf16's 64), the epilogue applies diag(sa) . diag(sb)
template <int BN, bool A_MN, bool B_MN, int EPI, int MSUB = 1, int CG = 1, bool F8 = false>
__global__ void __launch_bounds__(384, 1)
gemm_bf16_sm100(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const __grid_constant__ CUtensorMap tmO0, const __grid_constant__ CUtensorMap tmO1, GemmArgs g) {
    using C = GemmCfg<BN, MSUB, EPI, CG>;
    static_assert(CG == 1 || (MSUB == 1 && !A_MN && BN == 256 && EPI != EPI_F32), "CTA-pair GEMM shape");
    static_assert(!F8 || (!A_MN && !B_MN && MSUB == 1 && CG == 1 && EPI != EPI_F32), "FP8 GEMM shape");
    constexpr int KE = F8 ? 128 : C::BK;   // K elements per k-block
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = smem;
    uint8_t* sB = smem + C::STAGES * C::A_BYTES;
    uint8_t* stg = smem + C::STAGES * C::STAGE_BYTES;   // epilogue staging for the TMA stores
    uint64_t* full = reinterpret_cast<uint64_t*>(stg + C::STAGING);
    uint64_t* empty = full + C::STAGES;
    uint64_t* tfull = empty + C::STAGES;   // [2]
    uint64_t* tempty = tfull + 2;          // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x >> 5;
    const int total = g.m_tiles * g.n_tiles * g.k_splits;
    // CTA pairs: both CTAs walk the same tile sequence; rank 0 (leader) issues the MMAs
    const uint32_t rank = CG == 2 ? cluster_ctarank() : 0u;
    const int t_first = (int)blockIdx.x / CG, t_step = (int)gridDim.x / CG;

    if (threadIdx.x == 0) {
        // with fused column sums the 8 epilogue warps also read every B stage before it is released
        const int cs_arrivals = (EPI == EPI_F32 && g.colsum) ? 8 : 0;
        for (int i = 0; i < C::STAGES; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1 + cs_arrivals); }
        for (int i = 0; i < 2; ++i) { mbar_init(&tfull[i], 1); mbar_init(&tempty[i], 8 * CG); }
        fence_barrier_init();
    }
    if (warp == 0 && lane_id() == 0) { tma_prefetch_desc(&tmA); tma_prefetch_desc(&tmB); }
    if (warp == 2) {
        if (CG == 2) tmem_alloc_pair<C::TMEM_COLS>(tmem_slot);
        else tmem_alloc<C::TMEM_COLS>(tmem_slot);
    }
    tc_fence_before();
    __syncthreads();
    if (CG == 2) cluster_sync_all();   // the peer's barriers are initialised before any remote use
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    auto decode = [&](int t, int& mt, int& nt, int& ks) {
        ks = t / (g.m_tiles * g.n_tiles);
        int r = t - ks * g.m_tiles * g.n_tiles;
        mt = r / g.n_tiles;
        nt = r - mt * g.n_tiles;
    };
    auto kb_range = [&](int ks, int& kb0, int& kb1) {
        int nkb = (g.K + KE - 1) / KE;
        kb0 = ks * g.kb_per_split;
        kb1 = min(nkb, kb0 + g.kb_per_split);
    };

    if (warp == 0) {
        // ------------------------------------------------ TMA producer
        if (lane_id() == 0) {
            int stage = 0; uint32_t phase = 0;
            for (int t = t_first; t < total; t += t_step) {
                int mt, nt, ks, kb0, kb1;
                decode(t, mt, nt, ks);
                kb_range(ks, kb0, kb1);
                if (CG == 2) {   // this CTA's A rows and B columns; the follower counts on the leader's barrier
                    for (int kb = kb0; kb < kb1; ++kb) {
                        mbar_wait(&empty[stage], phase ^ 1);
                        uint8_t* a = sA + stage * C::A_BYTES;
                        uint8_t* b = sB + stage * C::B_BYTES;
                        const int arow = mt * 256 + (int)rank * 128, bcol = nt * BN + (int)rank * (BN / 2);
                        if (rank == 0) {
                            mbar_arrive_expect_tx(&full[stage], 2 * C::STAGE_BYTES);
                            tma_load_2d(a, &tmA, &full[stage], kb * KE, arow);
                            if (!B_MN) {
                                tma_load_2d(b, &tmB, &full[stage], kb * KE, bcol);
                            } else {
#pragma unroll
                                for (int j = 0; j < BN / 128; ++j)
                                    tma_load_2d(b + j * 64 * C::BK * 2, &tmB, &full[stage], bcol + j * 64, kb * KE);
                            }
                        } else {
                            const uint32_t lb = mapa_shared(smem_u32(&full[stage]), 0);
                            tma_load_2d_pair(a, &tmA, lb, kb * KE, arow);
                            if (!B_MN) {
                                tma_load_2d_pair(b, &tmB, lb, kb * KE, bcol);
                            } else {
#pragma unroll
                                for (int j = 0; j < BN / 128; ++j)
                                    tma_load_2d_pair(b + j * 64 * C::BK * 2, &tmB, lb, bcol + j * 64, kb * KE);
                            }
                        }
                        if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
                    }
                    continue;
                }
                for (int kb = kb0; kb < kb1; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    mbar_arrive_expect_tx(&full[stage], C::STAGE_BYTES);
                    uint8_t* a = sA + stage * C::A_BYTES;
                    uint8_t* b = sB + stage * C::B_BYTES;
                    if (!A_MN) {
                        tma_load_2d(a, &tmA, &full[stage], kb * KE, mt * C::BM);
                    } else {
#pragma unroll
                        for (int j = 0; j < C::BM / 64; ++j)
                            tma_load_2d(a + j * 64 * C::BK * 2, &tmA, &full[stage], mt * C::BM + j * 64, kb * KE);
                    }
                    if (!B_MN) {
                        tma_load_2d(b, &tmB, &full[stage], kb * KE, nt * BN);
                    } else {
#pragma unroll
                        for (int j = 0; j < BN / 64; ++j)
                            tma_load_2d(b + j * 64 * C::BK * 2, &tmB, &full[stage], nt * BN + j * 64, kb * KE);
                    }
                    if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1 && rank == 0) {
        // ------------------------------------------------ MMA issuer (CTA pairs: the leader, M = 256)
        constexpr uint32_t idesc = F8 ? make_idesc_e4m3(128, BN) : make_idesc_bf16(128 * CG, BN, A_MN, B_MN);
        int stage = 0; uint32_t phase = 0;
        int it = 0;
        for (int t = t_first; t < total; t += t_step, ++it) {
            int mt, nt, ks, kb0, kb1;
            decode(t, mt, nt, ks);
            kb_range(ks, kb0, kb1);
            const int acc = C::NACC == 2 ? (it & 1) : 0;
            mbar_wait(&tempty[acc], (C::NACC == 2 ? ((it >> 1) & 1) : (it & 1)) ^ 1);
            tc_fence_after();
            const uint32_t d_tmem = tmem_base + acc * MSUB * BN;
            // the next k-block's stage is probed (test_wait, never parks) before this block's MMAs
            // are issued and waited on after them: a blocking wait between blocks drains the MMA queue
            mbar_wait(&full[stage], phase);
            for (int kb = kb0; kb < kb1; ++kb) {
                tc_fence_after();
                const int nst = stage + 1 == C::STAGES ? 0 : stage + 1;
                const uint32_t nph = stage + 1 == C::STAGES ? phase ^ 1 : phase;
                const bool rdy = mbar_test(smem_u32(&full[nst]), nph);
                if (elect_one()) {
                    const uint32_t a0 = smem_u32(sA + stage * C::A_BYTES);
                    const uint32_t b0 = smem_u32(sB + stage * C::B_BYTES);
#pragma unroll
                    for (int k = 0; k < C::BK / 16; ++k) {
                        uint64_t bd = B_MN ? make_sw128_desc(b0 + k * 2048, 64 * C::BK * 2, 1024)
                                           : make_sw128_desc(b0 + k * 32, 16, 1024);
#pragma unroll
                        for (int ms = 0; ms < MSUB; ++ms) {   // rows [128 ms, 128 ms + 128) start 16 KB apart (both majors)
                            uint64_t ad = A_MN ? make_sw128_desc(a0 + ms * 16384 + k * 2048, 64 * C::BK * 2, 1024)
                                               : make_sw128_desc(a0 + ms * 16384 + k * 32, 16, 1024);
                            if (CG == 2) umma_ss_pair(d_tmem + ms * BN, ad, bd, idesc, (kb > kb0 || k > 0) ? 1u : 0u);
                            else if (F8) umma_ss_e4m3(d_tmem + ms * BN, ad, bd, idesc, (kb > kb0 || k > 0) ? 1u : 0u);
                            else umma_ss(d_tmem + ms * BN, ad, bd, idesc, (kb > kb0 || k > 0) ? 1u : 0u);
                        }
                    }
                    if (CG == 2) umma_commit_pair(&empty[stage]);
                    else umma_commit(&empty[stage]);
                }
                __syncwarp();
                stage = nst; phase = nph;
                if (kb + 1 < kb1 && !rdy) mbar_wait(&full[stage], phase);
            }
            if (elect_one()) {
                if (CG == 2) umma_commit_pair(&tfull[acc]);
                else umma_commit(&tfull[acc]);
            }
            __syncwarp();
        }
    } else if (warp >= 4) {
        // ------------------------------------------------ epilogue
        const int wq = warp & 3;              // TMEM lane quarter
        const int wg = (warp - 4) >> 2;       // column half of the tile
        const int row_in_tile = wq * 32 + (int)lane_id();
        int it = 0;
        int cs_stage = 0; uint32_t cs_phase = 0;   // B-stage sequence (mirrors the MMA issuer's)
        uint32_t n_chunk = 0;                      // TMA-store chunks this warp has staged
        const int row_base = CG == 2 ? (int)rank * 128 : 0;   // this CTA's half of a pair tile
        for (int t = t_first; t < total; t += t_step, ++it) {
            int mt, nt, ks;
            decode(t, mt, nt, ks);
            if (EPI == EPI_F32 && B_MN && BN == 256 && g.colsum) {
                // bias gradient = column sums of B, read from the staged k-blocks (m-tile 0 only, so
                // each B element is counted once): thread -> 8 columns x 8 rows of every stage
                const int et = threadIdx.x - 128, c = et & 31, r = et >> 5;
                float cs[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) cs[e] = 0.f;
                int kb0, kb1;
                kb_range(ks, kb0, kb1);
                for (int kb = kb0; kb < kb1; ++kb) {
                    mbar_wait(&full[cs_stage], cs_phase);
                    if (mt == 0) {
                        const uint8_t* b = sB + cs_stage * C::B_BYTES + (c >> 3) * (64 * C::BK * 2);
#pragma unroll
                        for (int rr = 0; rr < 8; ++rr) {
                            const int k = r * 8 + rr;
                            const uint4 u = *reinterpret_cast<const uint4*>(b + k * 128 + (((c & 7) ^ rr) << 4));
                            const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
                            for (int q = 0; q < 4; ++q) {
                                const float2 f = unpack_bf16x2(w[q]);
                                cs[2 * q] += f.x;
                                cs[2 * q + 1] += f.y;
                            }
                        }
                    }
                    __syncwarp();
                    if (lane_id() == 0) mbar_arrive(&empty[cs_stage]);
                    if (++cs_stage == C::STAGES) { cs_stage = 0; cs_phase ^= 1; }
                }
                if (mt == 0) {
                    float* red = reinterpret_cast<float*>(stg);   // [8 row groups][BN]
#pragma unroll
                    for (int e = 0; e < 8; ++e) red[r * BN + c * 8 + e] = cs[e];
                    named_bar_sync(1, 256);
                    float sum = 0.f;
#pragma unroll
                    for (int q = 0; q < 8; ++q) sum += red[q * BN + et];
                    const int col = nt * BN + et;
                    if (col < g.N && sum != 0.f) atomicAdd(g.colsum + col, sum);
                    named_bar_sync(1, 256);
                }
            }
            // this warp's bias columns, one per lane per 32-column chunk, loaded before the
            // accumulator wait (their latency hides behind the main loop); broadcast by shuffles
            constexpr int NCH = BN / 64;   // 32-column chunks per warpgroup half
            float bl[NCH];
#pragma unroll
            for (int q = 0; q < NCH; ++q) {
                const int cb = nt * BN + wg * (BN / 2) + 32 * q + (int)lane_id();
                bl[q] = (EPI != EPI_F32 && g.bias && cb < g.N) ? __ldg(g.bias + cb) * (EPI == EPI_SILU ? 0.5f : 1.0f) : 0.f;
            }
            float sbl[F8 ? NCH : 1];   // F8: this warp's column scales, one per lane per chunk (x 1/2 for SiLU's h/2)
#pragma unroll
            for (int q = 0; q < (F8 ? NCH : 1); ++q) {
                const int cb = nt * BN + wg * (BN / 2) + 32 * q + (int)lane_id();
                sbl[q] = (F8 && cb < g.N) ? __ldg(g.scale_b + cb) * (EPI == EPI_SILU ? 0.5f : 1.0f) : 0.f;
            }
            const int acc = C::NACC == 2 ? (it & 1) : 0;
            mbar_wait(&tfull[acc], C::NACC == 2 ? ((it >> 1) & 1) : (it & 1));
            tc_fence_after();
#pragma unroll 1
            for (int ms = 0; ms < MSUB; ++ms) {
            const int row = mt * C::BM * CG + row_base + ms * 128 + row_in_tile;
            const bool row_ok = row < g.M;
            const float sa_row = (F8 && row_ok) ? __ldg(g.scale_a + row) : 0.f;
#pragma unroll 1
            for (int c0 = wg * (BN / 2); c0 < (wg + 1) * (BN / 2); c0 += 32) {
                float v[32];
                const int col = nt * BN + c0;
                // residual row segment (64 B) requested before the accumulator load: the two latencies overlap
                uint4 rv4[4];
                const bool use_res = EPI == EPI_BF16 && g.resid && row_ok && col < g.N;
                if (use_res) {
                    const uint4* rp = reinterpret_cast<const uint4*>(g.resid + (int64_t)row * g.ldr + col);
#pragma unroll
                    for (int j = 0; j < 4; ++j) rv4[j] = __ldg(rp + j);
                }
                tmem_ld32(tmem_base + ((uint32_t)(wq * 32) << 16) + (acc * MSUB + ms) * BN + c0, v);
                tmem_ld_wait();
                if (col >= g.N) continue;   // warp-uniform
                if (EPI == EPI_F32) {
                    if (!row_ok) continue;
                    float* o = reinterpret_cast<float*>(g.out0) + (int64_t)row * g.ld0 + col;
#pragma unroll
                    for (int j = 0; j < 32; j += 4)
                        atomicAdd(reinterpret_cast<float4*>(o + j), make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]));
                } else {
                    // h = acc + bias (EPI_SILU: h/2 carried, silu(2h') = h' + h' tanh h'); packed bf16
                    float hb[32];
                    {
                        const int q = (c0 - wg * (BN / 2)) >> 5;   // chunk index within the half
                        float bq = bl[0];
#pragma unroll
                        for (int qq = 1; qq < NCH; ++qq) bq = q == qq ? bl[qq] : bq;
#pragma unroll
                        for (int j = 0; j < 32; ++j) hb[j] = __shfl_sync(0xffffffffu, bq, j);
                    }
                    if (F8) {   // acc x sa x sb: the SiLU's 1/2 rides in sb, so the epilogues below see 1/2 -> 1
                        const int q = (c0 - wg * (BN / 2)) >> 5;
                        float sq = sbl[0];
#pragma unroll
                        for (int qq = 1; qq < (F8 ? NCH : 1); ++qq) sq = q == qq ? sbl[qq] : sq;
#pragma unroll
                        for (int j = 0; j < 32; ++j) v[j] *= sa_row * __shfl_sync(0xffffffffu, sq, j);
                    }
                    uint32_t o0[16], o1[16];
                    if (EPI == EPI_BF16) {
#pragma unroll
                        for (int j = 0; j < 32; ++j) v[j] += hb[j];
                        if (use_res) {
#pragma unroll
                            for (int j = 0; j < 4; ++j) {
                                const __nv_bfloat162* r2 = reinterpret_cast<const __nv_bfloat162*>(&rv4[j]);
#pragma unroll
                                for (int e = 0; e < 4; ++e) {
                                    float2 f = __bfloat1622float2(r2[e]);
                                    v[j * 8 + 2 * e] += f.x;
                                    v[j * 8 + 2 * e + 1] += f.y;
                                }
                            }
                        }
#pragma unroll
                        for (int i = 0; i < 16; ++i) o0[i] = pack_bf16(v[2 * i], v[2 * i + 1]);
                    } else {  // EPI_SILU (packed fp32): silu = h + h t;  silu' = (1 + t)(1 + h (1 - t)) / 2;  h = acc/2, t = tanh h
                        const uint64_t half2 = f2_pack(0.5f, 0.5f), one2 = f2_pack(1.f, 1.f), neg2 = f2_pack(-1.f, -1.f);
#pragma unroll
                        for (int i = 0; i < 16; ++i) {
                            const uint64_t H = ffma2(f2_pack(v[2 * i], v[2 * i + 1]), F8 ? one2 : half2, f2_pack(hb[2 * i], hb[2 * i + 1]));
                            const float2 hh = f2_unpack(H);
                            const uint64_t T = f2_pack(tanh_approx(hh.x), tanh_approx(hh.y));
                            const float2 sv = f2_unpack(ffma2(H, T, H));
                            o0[i] = pack_bf16(sv.x, sv.y);
                            if (g.out1) {
                                const float2 gv = f2_unpack(fmul2(ffma2(T, half2, half2), ffma2(H, ffma2(T, neg2, one2), one2)));
                                o1[i] = pack_bf16(gv.x, gv.y);
                            }
                        }
                    }
                    // rows of this warp -> its 64B-swizzled 32x32 staging boxes -> TMA stores
                    // (coalesced; rows / columns beyond M, N are clipped by the tensor map)
                    // one output: the two 2 KB boxes alternate chunk by chunk, so a chunk's staging
                    // overlaps the previous chunk's TMA read (wait for all but the newest group);
                    // two outputs: box0 / box1 per chunk, all previous stores read first
                    const bool dbuf = !(EPI == EPI_SILU && g.out1);
                    uint8_t* box0 = stg + (warp - 4) * 4096 + (dbuf && (n_chunk & 1) ? 2048 : 0);
                    uint8_t* box1 = stg + (warp - 4) * 4096 + 2048;
                    ++n_chunk;
                    if (lane_id() == 0) { if (dbuf) bulk_wait_read1(); else bulk_wait_read0(); }
                    __syncwarp();
                    const int r = lane_id();
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        const int off = r * 64 + ((c ^ ((r >> 1) & 3)) << 4);
                        *reinterpret_cast<uint4*>(box0 + off) = make_uint4(o0[4 * c], o0[4 * c + 1], o0[4 * c + 2], o0[4 * c + 3]);
                        if (EPI == EPI_SILU && g.out1)
                            *reinterpret_cast<uint4*>(box1 + off) = make_uint4(o1[4 * c], o1[4 * c + 1], o1[4 * c + 2], o1[4 * c + 3]);
                    }
                    fence_proxy_async_smem();
                    __syncwarp();
                    if (lane_id() == 0) {
                        const int row0 = mt * C::BM * CG + row_base + ms * 128 + wq * 32;
                        tma_store_2d(&tmO0, box0, col, row0);
                        if (EPI == EPI_SILU && g.out1) tma_store_2d(&tmO1, box1, col, row0);
                        bulk_commit();
                    }
                }
            }
            }   // ms
            tc_fence_before();
            __syncwarp();
            if (lane_id() == 0) {
                if (CG == 2 && rank != 0) mbar_arrive_cluster(mapa_shared(smem_u32(&tempty[acc]), 0));
                else mbar_arrive(&tempty[acc]);
            }
        }
    }
    if (warp >= 4 && lane_id() == 0) bulk_wait0();   // TMA stores complete before the CTA retires
    __syncthreads();
    if (CG == 2) {
        cluster_sync_all();   // both CTAs done with the pair's TMEM
        if (warp == 2) tmem_dealloc_pair<C::TMEM_COLS>(tmem_base);
    } else if (warp == 2) {
        tmem_dealloc<C::TMEM_COLS>(tmem_base);
    }
}

}  // namespace uh
