// gemm.cu — launchers for the projection GEMMs: the tcgen05 bf16 kernel
// (gemm_sm100.cuh) and the fp32 SIMT verification twin.
#include <algorithm>

#include "gemm_sm100.cuh"
#include <cstdlib>

#include "internal.h"

namespace uh {

// ============================================================== fp32 SIMT twin
// C[m,n] = sum_k A(m,k) B(k,n); 64x64 tile, 16-deep K slab, 256 threads, 4x4 per thread.
template <int EPI>
__global__ void __launch_bounds__(256) gemm_f32_simt(int M, int N, int K, const float* __restrict__ A, int64_t sam,
                                                      int64_t sak, const float* __restrict__ B, int64_t sbk, int64_t sbn,
                                                      float* out0, int64_t ld0, float* out1, int64_t ld1,
                                                      const float* __restrict__ bias, const float* __restrict__ resid,
                                                      int64_t ldr, int kchunk) {
    __shared__ float As[16][64 + 1];
    __shared__ float Bs[16][64 + 1];
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int m0 = blockIdx.y * 64, n0 = blockIdx.x * 64;
    const int kbeg = blockIdx.z * kchunk, kend = min(K, kbeg + kchunk);
    float acc[4][4] = {};
    for (int k0 = kbeg; k0 < kend; k0 += 16) {
        for (int i = threadIdx.x; i < 16 * 64; i += 256) {
            int kk = i / 64, mm = i % 64;
            int gm = m0 + mm, gk = k0 + kk;
            As[kk][mm] = (gm < M && gk < kend) ? A[gm * sam + gk * sak] : 0.f;
            int gn = n0 + mm;
            Bs[kk][mm] = (gn < N && gk < kend) ? B[gk * sbk + gn * sbn] : 0.f;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < 16; ++kk) {
            float a[4], b[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) { a[i] = As[kk][ty * 4 + i]; b[i] = Bs[kk][tx * 4 + i]; }
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        int m = m0 + ty * 4 + i;
        if (m >= M) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            int n = n0 + tx * 4 + j;
            if (n >= N) continue;
            float v = acc[i][j];
            if (EPI == EPI_F32) { atomicAdd(out0 + m * ld0 + n, v); continue; }
            if (bias) v += bias[n];
            if (EPI == EPI_BF16) {
                if (resid) v += resid[m * ldr + n];
                out0[m * ld0 + n] = v;
            } else {
                float sg = 1.0f / (1.0f + expf(-v));
                out0[m * ld0 + n] = v * sg;
                if (out1) out1[m * ld1 + n] = sg * (1.0f + v * (1.0f - sg));
            }
        }
    }
}

static uh_status gemm_f32(const GemmDesc& g, cudaStream_t st) {
    // element (m,k) of A and (k,n) of B as strides
    int64_t sam = g.a_mn ? 1 : g.lda, sak = g.a_mn ? g.lda : 1;
    int64_t sbk = g.b_mn ? g.ldb : 1, sbn = g.b_mn ? 1 : g.ldb;
    int splits = 1, kchunk = g.K;
    if (g.epi == EPI_F32) {
        int tiles = ((g.M + 63) / 64) * ((g.N + 63) / 64);
        splits = std::max(1, std::min((g.K + 255) / 256, (2 * num_sms() + tiles - 1) / tiles));
        kchunk = ((g.K + splits - 1) / splits + 15) / 16 * 16;
        splits = (g.K + kchunk - 1) / kchunk;
    }
    dim3 grid((g.N + 63) / 64, (g.M + 63) / 64, std::max(splits, 1));
    const float* A = (const float*)g.A;
    const float* B = (const float*)g.B;
    if (g.M == 0 || g.N == 0) return UH_OK;
    if (g.K == 0 && g.epi == EPI_F32) return UH_OK;
    switch (g.epi) {
        case EPI_BF16:
            gemm_f32_simt<EPI_BF16><<<grid, 256, 0, st>>>(g.M, g.N, g.K, A, sam, sak, B, sbk, sbn, (float*)g.out0, g.ld0,
                                                         (float*)g.out1, g.ld1, g.bias, (const float*)g.resid, g.ldr, kchunk);
            note_launch();
            break;
        case EPI_SILU:
            gemm_f32_simt<EPI_SILU><<<grid, 256, 0, st>>>(g.M, g.N, g.K, A, sam, sak, B, sbk, sbn, (float*)g.out0, g.ld0,
                                                         (float*)g.out1, g.ld1, g.bias, (const float*)g.resid, g.ldr, kchunk);
            note_launch();
            break;
        default:
            gemm_f32_simt<EPI_F32><<<grid, 256, 0, st>>>(g.M, g.N, g.K, A, sam, sak, B, sbk, sbn, (float*)g.out0, g.ld0,
                                                        (float*)g.out1, g.ld1, g.bias, (const float*)g.resid, g.ldr, kchunk);
            note_launch();
    }
    UH_CUDA(cudaGetLastError());
    return UH_OK;
}

// ============================================================== bf16 tcgen05
template <int BN, bool AMN, bool BMN, int EPI, int MSUB = 1, int CG = 1>
static uh_status launch_sm100(const GemmDesc& g, cudaStream_t st) {
    using C = GemmCfg<BN, MSUB, EPI, CG>;
    CUtensorMap ta, tb;
    if (!AMN) UH_TRY(make_tmap_bf16(&ta, g.A, g.K, g.M, g.lda, 64, C::BM));
    else      UH_TRY(make_tmap_bf16(&ta, g.A, g.M, g.K, g.lda, 64, 64));
    if (!BMN) UH_TRY(make_tmap_bf16(&tb, g.B, g.K, g.N, g.ldb, 64, BN / CG));   // CTA pairs: each CTA its BN/2 rows
    else      UH_TRY(make_tmap_bf16(&tb, g.B, g.N, g.K, g.ldb, 64, 64));
    // outputs leave through TMA stores of 32x32 boxes (64B swizzle, matching the staging layout)
    CUtensorMap to0 = ta, to1 = ta;
    if (EPI != EPI_F32) {
        UH_TRY(make_tmap_bf16(&to0, g.out0, g.N, g.M, g.ld0, 32, 32, 64));
        if (g.out1) UH_TRY(make_tmap_bf16(&to1, g.out1, g.N, g.M, g.ld1, 32, 32, 64));
    }
    GemmArgs a;
    a.M = g.M; a.N = g.N; a.K = g.K;
    a.m_tiles = (g.M + C::BM * CG - 1) / (C::BM * CG);
    a.n_tiles = (g.N + BN - 1) / BN;
    const int nkb = (g.K + C::BK - 1) / C::BK;
    const int sms = num_sms();
    int splits = 1;
    if (EPI == EPI_F32) {   // split-K: one wave (tiles x splits <= SMs; a partial second wave doubles the critical path)
        const int tiles = a.m_tiles * a.n_tiles;
        splits = std::max(1, std::min(nkb, sms / std::max(1, tiles)));
    }
    a.kb_per_split = (nkb + splits - 1) / splits;
    a.k_splits = (nkb + a.kb_per_split - 1) / a.kb_per_split;
    a.out0 = g.out0; a.ld0 = g.ld0; a.out1 = g.out1; a.ld1 = g.ld1;
    a.bias = g.bias; a.resid = (const __nv_bfloat16*)g.resid; a.ldr = g.ldr;
    a.colsum = (EPI == EPI_F32 && BMN && BN == 256) ? g.colsum : nullptr;
    const int total = a.m_tiles * a.n_tiles * a.k_splits;
    auto kern = gemm_bf16_sm100<BN, AMN, BMN, EPI, MSUB, CG>;
    UH_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    if (CG == 2) {   // CTA pairs: a cluster of two per pair tile
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)(2 * std::min(total, sms / 2)));
        cfg.blockDim = dim3(384);
        cfg.dynamicSmemBytes = C::SMEM;
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 2; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        UH_CUDA(cudaLaunchKernelEx(&cfg, kern, ta, tb, to0, to1, a));
    } else {
        kern<<<std::min(total, sms), 384, C::SMEM, st>>>(ta, tb, to0, to1, a);
    }
    note_launch();
    UH_CUDA(cudaGetLastError());
    return UH_OK;
}

// ============================================================== E4M3 tcgen05 (NEXT-2)
template <int BN, int EPI>
static uh_status launch_fp8(const GemmDesc& g, const float* sa, const float* sb, cudaStream_t st) {
    using C = GemmCfg<BN, 1, EPI, 1>;
    CUtensorMap ta, tb, to0, to1;
    UH_TRY(make_tmap_u8(&ta, g.A, g.K, g.M, g.lda, 128, C::BM));    // [M][K] codes, 128-byte K rows
    UH_TRY(make_tmap_u8(&tb, g.B, g.K, g.N, g.ldb, 128, BN));       // B^T [N][K]
    UH_TRY(make_tmap_bf16(&to0, g.out0, g.N, g.M, g.ld0, 32, 32, 64));
    to1 = to0;
    if (g.out1) UH_TRY(make_tmap_bf16(&to1, g.out1, g.N, g.M, g.ld1, 32, 32, 64));
    GemmArgs a;
    a.M = g.M; a.N = g.N; a.K = g.K;
    a.m_tiles = (g.M + C::BM - 1) / C::BM;
    a.n_tiles = (g.N + BN - 1) / BN;
    a.kb_per_split = (g.K + 127) / 128;
    a.k_splits = 1;
    a.out0 = g.out0; a.ld0 = g.ld0; a.out1 = g.out1; a.ld1 = g.ld1;
    a.bias = g.bias; a.resid = (const __nv_bfloat16*)g.resid; a.ldr = g.ldr;
    a.colsum = nullptr;
    a.scale_a = sa; a.scale_b = sb;
    const int total = a.m_tiles * a.n_tiles;
    auto kern = gemm_bf16_sm100<BN, false, false, EPI, 1, 1, true>;
    UH_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    kern<<<std::min(total, num_sms()), 384, C::SMEM, st>>>(ta, tb, to0, to1, a);
    note_launch();
    UH_CUDA(cudaGetLastError());
    return UH_OK;
}

uh_status gemm_fp8_run(const GemmDesc& g, const float* sa, const float* sb, cudaStream_t st) {
    if (g.M == 0 || g.N == 0) return UH_OK;
    if (g.K <= 0 || g.K % 128) return fail(UH_ERR_UNSUPPORTED, "fp8 gemm needs K % 128 == 0");
    if (g.N % 128) return fail(UH_ERR_UNSUPPORTED, "fp8 gemm needs N % 128 == 0");
    if (g.a_mn || g.b_mn) return fail(UH_ERR_UNSUPPORTED, "fp8 gemm operands are K-major");
    if (g.epi == EPI_SILU) {
        if (g.N % 256 == 0) return launch_fp8<256, EPI_SILU>(g, sa, sb, st);
        return launch_fp8<128, EPI_SILU>(g, sa, sb, st);
    }
    if (g.epi == EPI_BF16) {
        if (g.N % 256 == 0) return launch_fp8<256, EPI_BF16>(g, sa, sb, st);
        return launch_fp8<128, EPI_BF16>(g, sa, sb, st);
    }
    return fail(UH_ERR_UNSUPPORTED, "fp8 gemm epilogue");
}

uh_status gemm_run(const GemmDesc& g, uh_dtype dt, cudaStream_t st) {
    if (g.M == 0 || g.N == 0) return UH_OK;
    if (g.K == 0) return g.epi == EPI_F32 ? UH_OK : fail(UH_ERR_UNSUPPORTED, "gemm with K == 0");
    if (dt == UH_F32) return gemm_f32(g, st);
    // bf16: N must be a multiple of 64 (checked by callers: d = 128 * H)
    const bool wide = g.N % 256 == 0 && g.epi != EPI_F32;
#define UH_G(BN, AM, BM_, E) return launch_sm100<BN, AM, BM_, E>(g, st)
    if (g.epi == EPI_F32) {
        // weight gradients (K = tokens): 256 x 256 tiles (two 128-row sub-tiles share each B k-block)
        if (g.a_mn && g.b_mn && g.M % 256 == 0 && g.N % 256 == 0) return launch_sm100<256, true, true, EPI_F32, 2>(g, st);
        if (g.colsum) return fail(UH_ERR_UNSUPPORTED, "fused column sums need the 256-wide split-K path");
        if (g.a_mn && g.b_mn) UH_G(128, true, true, EPI_F32);
        if (!g.a_mn && !g.b_mn) UH_G(128, false, false, EPI_F32);
        return fail(UH_ERR_UNSUPPORTED, "gemm EPI_F32 with mixed majors");
    }
    if (g.a_mn) return fail(UH_ERR_UNSUPPORTED, "gemm bf16-out with MN-major A");
    // CTA pairs (cta_group::2, 256 x 256 pair tiles) for the K-major-A projections: g.pair = 1
    // enables them for MN-major B (f1, f2), 2 for both B majors (also dY).  The layer leaves
    // g.pair at kGemmPairDefault (off: measured equal to single CTAs at cfg3,
    // profiles/r01_gemm_pair_ab.log); the test hook exercises both.
    const bool pair = wide && (g.pair >= 2 || (g.pair == 1 && g.b_mn));
    if (g.epi == EPI_SILU) {
        if (pair) {
            if (g.b_mn) return launch_sm100<256, false, true, EPI_SILU, 1, 2>(g, st);
            return launch_sm100<256, false, false, EPI_SILU, 1, 2>(g, st);
        }
        if (wide) { if (g.b_mn) UH_G(256, false, true, EPI_SILU); UH_G(256, false, false, EPI_SILU); }
        if (g.b_mn) UH_G(128, false, true, EPI_SILU);
        UH_G(128, false, false, EPI_SILU);
    }
    // long K (dx^ = dH W1^T, K = 4d): 256 x 256 tiles of two 128-row sub-tiles halve the B ingress
    // per flop; the single accumulator's unoverlapped epilogue is small against the K loop
    if (wide && g.K >= 1024 && g.M % 256 == 0 && !g.resid) {
        if (g.b_mn) return launch_sm100<256, false, true, EPI_BF16, 2>(g, st);
        return launch_sm100<256, false, false, EPI_BF16, 2>(g, st);
    }
    if (pair && g.K < 1024) {
        if (g.b_mn) return launch_sm100<256, false, true, EPI_BF16, 1, 2>(g, st);
        return launch_sm100<256, false, false, EPI_BF16, 1, 2>(g, st);
    }
    if (wide) { if (g.b_mn) UH_G(256, false, true, EPI_BF16); UH_G(256, false, false, EPI_BF16); }
    if (g.b_mn) UH_G(128, false, true, EPI_BF16);
    UH_G(128, false, false, EPI_BF16);
#undef UH_G
}

}  // namespace uh
