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
};

template <int BN>
struct GemmCfg {
    static constexpr int BM = 128, BK = 64;
    static constexpr int STAGES = BN == 256 ? 4 : 6;
    static constexpr int A_BYTES = BM * BK * 2;
    static constexpr int B_BYTES = BN * BK * 2;
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
    static constexpr int TMEM_COLS = 2 * BN <= 256 ? 256 : 512;
};

template <int BN, bool A_MN, bool B_MN, int EPI>
__global__ void __launch_bounds__(384, 1)
gemm_bf16_sm100(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, GemmArgs g) {
    using C = GemmCfg<BN>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = smem;
    uint8_t* sB = smem + C::STAGES * C::A_BYTES;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE_BYTES);
    uint64_t* empty = full + C::STAGES;
    uint64_t* tfull = empty + C::STAGES;   // [2]
    uint64_t* tempty = tfull + 2;          // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x >> 5;
    const int total = g.m_tiles * g.n_tiles * g.k_splits;

    if (threadIdx.x == 0) {
        for (int i = 0; i < C::STAGES; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
        for (int i = 0; i < 2; ++i) { mbar_init(&tfull[i], 1); mbar_init(&tempty[i], 8); }
        fence_barrier_init();
    }
    if (warp == 0 && lane_id() == 0) { tma_prefetch_desc(&tmA); tma_prefetch_desc(&tmB); }
    if (warp == 2) tmem_alloc<C::TMEM_COLS>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    auto decode = [&](int t, int& mt, int& nt, int& ks) {
        ks = t / (g.m_tiles * g.n_tiles);
        int r = t - ks * g.m_tiles * g.n_tiles;
        mt = r / g.n_tiles;
        nt = r - mt * g.n_tiles;
    };
    auto kb_range = [&](int ks, int& kb0, int& kb1) {
        int nkb = (g.K + C::BK - 1) / C::BK;
        kb0 = ks * g.kb_per_split;
        kb1 = min(nkb, kb0 + g.kb_per_split);
    };

    if (warp == 0) {
        // ------------------------------------------------ TMA producer
        if (lane_id() == 0) {
            int stage = 0; uint32_t phase = 0;
            for (int t = blockIdx.x; t < total; t += gridDim.x) {
                int mt, nt, ks, kb0, kb1;
                decode(t, mt, nt, ks);
                kb_range(ks, kb0, kb1);
                for (int kb = kb0; kb < kb1; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    mbar_arrive_expect_tx(&full[stage], C::STAGE_BYTES);
                    uint8_t* a = sA + stage * C::A_BYTES;
                    uint8_t* b = sB + stage * C::B_BYTES;
                    if (!A_MN) {
                        tma_load_2d(a, &tmA, &full[stage], kb * C::BK, mt * C::BM);
                    } else {
#pragma unroll
                        for (int j = 0; j < C::BM / 64; ++j)
                            tma_load_2d(a + j * 64 * C::BK * 2, &tmA, &full[stage], mt * C::BM + j * 64, kb * C::BK);
                    }
                    if (!B_MN) {
                        tma_load_2d(b, &tmB, &full[stage], kb * C::BK, nt * BN);
                    } else {
#pragma unroll
                        for (int j = 0; j < BN / 64; ++j)
                            tma_load_2d(b + j * 64 * C::BK * 2, &tmB, &full[stage], nt * BN + j * 64, kb * C::BK);
                    }
                    if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------ MMA issuer
        constexpr uint32_t idesc = make_idesc_bf16(C::BM, BN, A_MN, B_MN);
        int stage = 0; uint32_t phase = 0;
        int it = 0;
        for (int t = blockIdx.x; t < total; t += gridDim.x, ++it) {
            int mt, nt, ks, kb0, kb1;
            decode(t, mt, nt, ks);
            kb_range(ks, kb0, kb1);
            const int acc = it & 1;
            mbar_wait(&tempty[acc], ((it >> 1) & 1) ^ 1);
            tc_fence_after();
            const uint32_t d_tmem = tmem_base + acc * BN;
            for (int kb = kb0; kb < kb1; ++kb) {
                mbar_wait(&full[stage], phase);
                tc_fence_after();
                if (elect_one()) {
                    const uint32_t a0 = smem_u32(sA + stage * C::A_BYTES);
                    const uint32_t b0 = smem_u32(sB + stage * C::B_BYTES);
#pragma unroll
                    for (int k = 0; k < C::BK / 16; ++k) {
                        uint64_t ad = A_MN ? make_sw128_desc(a0 + k * 2048, 64 * C::BK * 2, 1024)
                                           : make_sw128_desc(a0 + k * 32, 16, 1024);
                        uint64_t bd = B_MN ? make_sw128_desc(b0 + k * 2048, 64 * C::BK * 2, 1024)
                                           : make_sw128_desc(b0 + k * 32, 16, 1024);
                        umma_ss(d_tmem, ad, bd, idesc, (kb > kb0 || k > 0) ? 1u : 0u);
                    }
                    umma_commit(&empty[stage]);
                }
                __syncwarp();
                if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
            }
            if (elect_one()) umma_commit(&tfull[acc]);
            __syncwarp();
        }
    } else if (warp >= 4) {
        // ------------------------------------------------ epilogue
        const int wq = warp & 3;              // TMEM lane quarter
        const int wg = (warp - 4) >> 2;       // column half of the tile
        const int row_in_tile = wq * 32 + (int)lane_id();
        int it = 0;
        for (int t = blockIdx.x; t < total; t += gridDim.x, ++it) {
            int mt, nt, ks;
            decode(t, mt, nt, ks);
            const int acc = it & 1;
            mbar_wait(&tfull[acc], (it >> 1) & 1);
            tc_fence_after();
            const int row = mt * C::BM + row_in_tile;
            const bool row_ok = row < g.M;
#pragma unroll 1
            for (int c0 = wg * (BN / 2); c0 < (wg + 1) * (BN / 2); c0 += 32) {
                float v[32];
                tmem_ld32(tmem_base + ((uint32_t)(wq * 32) << 16) + acc * BN + c0, v);
                tmem_ld_wait();
                const int col = nt * BN + c0;
                if (!row_ok || col >= g.N) continue;
                if (EPI == EPI_F32) {
                    float* o = reinterpret_cast<float*>(g.out0) + (int64_t)row * g.ld0 + col;
#pragma unroll
                    for (int j = 0; j < 32; j += 4)
                        atomicAdd(reinterpret_cast<float4*>(o + j), make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]));
                } else {
                    if (g.bias) {
#pragma unroll
                        for (int j = 0; j < 32; ++j) v[j] += __ldg(g.bias + col + j);
                    }
                    if (EPI == EPI_BF16) {
                        if (g.resid) {
                            const uint4* rp = reinterpret_cast<const uint4*>(g.resid + (int64_t)row * g.ldr + col);
#pragma unroll
                            for (int j = 0; j < 4; ++j) {
                                uint4 rv = __ldg(rp + j);
                                const __nv_bfloat162* r2 = reinterpret_cast<const __nv_bfloat162*>(&rv);
#pragma unroll
                                for (int e = 0; e < 4; ++e) {
                                    float2 f = __bfloat1622float2(r2[e]);
                                    v[j * 8 + 2 * e] += f.x;
                                    v[j * 8 + 2 * e + 1] += f.y;
                                }
                            }
                        }
                        uint4* op = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(g.out0) + (int64_t)row * g.ld0 + col);
#pragma unroll
                        for (int j = 0; j < 4; ++j)
                            op[j] = make_uint4(pack_bf16(v[j * 8 + 0], v[j * 8 + 1]), pack_bf16(v[j * 8 + 2], v[j * 8 + 3]),
                                               pack_bf16(v[j * 8 + 4], v[j * 8 + 5]), pack_bf16(v[j * 8 + 6], v[j * 8 + 7]));
                    } else {  // EPI_SILU
                        // silu(v) = h (1 + t), silu'(v) = (1 + t)(1 + h (1 - t)) / 2, h = v/2, t = tanh(h)
                        float s[32], gp[32];
#pragma unroll
                        for (int j = 0; j < 32; ++j) {
                            const float hv = 0.5f * v[j];
                            const float t = tanh_approx(hv);
                            s[j] = fmaf(hv, t, hv);
                            gp[j] = 0.5f * (1.0f + t) * fmaf(hv, 1.0f - t, 1.0f);
                        }
                        uint4* op = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(g.out0) + (int64_t)row * g.ld0 + col);
#pragma unroll
                        for (int j = 0; j < 4; ++j)
                            op[j] = make_uint4(pack_bf16(s[j * 8 + 0], s[j * 8 + 1]), pack_bf16(s[j * 8 + 2], s[j * 8 + 3]),
                                               pack_bf16(s[j * 8 + 4], s[j * 8 + 5]), pack_bf16(s[j * 8 + 6], s[j * 8 + 7]));
                        if (g.out1) {
                            uint4* gq = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(g.out1) + (int64_t)row * g.ld1 + col);
#pragma unroll
                            for (int j = 0; j < 4; ++j)
                                gq[j] = make_uint4(pack_bf16(gp[j * 8 + 0], gp[j * 8 + 1]), pack_bf16(gp[j * 8 + 2], gp[j * 8 + 3]),
                                                   pack_bf16(gp[j * 8 + 4], gp[j * 8 + 5]), pack_bf16(gp[j * 8 + 6], gp[j * 8 + 7]));
                        }
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane_id() == 0) mbar_arrive(&tempty[acc]);
        }
    }
    __syncthreads();
    if (warp == 2) tmem_dealloc<C::TMEM_COLS>(tmem_base);
}

}  // namespace uh
