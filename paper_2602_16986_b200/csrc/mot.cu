// mot.cu — NEXT-4: the Mixture of Transducers fusion (include/uhstu_mot.h; arXiv 2602.16986
// §4.3, App. A; readings R28-R30 of DESIGN.md).
//
//   Z = [X_0[cand] | ... | X_{K-1}[cand]]  (candidate gather, one warp per (candidate, branch) row)
//   E = Z W_f + b_f                        (tcgen05 GEMM, bias epilogue)
//   dZ = dE W_f^T -> dX_k[cand]            (GEMM, then the inverse scatter over zeroed dX_k)
//   dW_f = Z^T dE, db_f = colsum(dE)        (split-K fp32 GEMM, column sums fused when 256-wide)
//
// The candidate rows come from the device offsets inside the kernels, so one launch covers
// every branch and user; the gather / scatter are HBM-bound row copies (16-byte vectors).
#include <algorithm>
#include <string>

#include "../../include/uhstu_mot.h"
#include "gemm_sm100.cuh"  // EPI_* constants
#include "internal.h"

namespace uh {
namespace {

constexpr int kMaxBranches = 8;

struct MotRows {
    uint8_t* x[kMaxBranches];            // branch rows (X_k for the gather, dX_k for the scatter)
    int64_t ld_bytes[kMaxBranches];
    const int32_t* off[kMaxBranches];    // device offsets of branch k
    int n;                               // branches
};

// row of candidate c = b n_cand + j in branch k: offsets_k[b + 1] - n_cand + j (R29)
__device__ __forceinline__ int64_t cand_row(const int32_t* off, int64_t c, int n_cand) {
    const int64_t b = c / n_cand;
    return (int64_t)__ldg(off + b + 1) - n_cand + (c - b * n_cand);
}

// SCATTER = false: Z[c, k row_bytes ...] = X_k[cand_row];  true: X_k[cand_row] = Z[c, k row_bytes ...]
template <bool SCATTER>
__global__ void __launch_bounds__(256) mot_rows_k(const __grid_constant__ MotRows br, int64_t C, int n_cand,
                                                  int64_t row_bytes, uint8_t* __restrict__ z, int64_t ldz_bytes) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * 8, n = C * br.n, nvec = row_bytes / 16;
    for (int64_t i = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5); i < n; i += warps) {
        const int k = (int)(i % br.n);
        const int64_t c = i / br.n;
        uint4* xr = reinterpret_cast<uint4*>(br.x[k] + cand_row(br.off[k], c, n_cand) * br.ld_bytes[k]);
        uint4* zr = reinterpret_cast<uint4*>(z + c * ldz_bytes + k * row_bytes);
        for (int64_t v = lane; v < nvec; v += 32) {
            if (SCATTER) xr[v] = zr[v]; else zr[v] = __ldg(xr + v);
        }
    }
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }
size_t round256(size_t b) { return (b + 255) & ~size_t(255); }

struct MotShape {
    int64_t C = 0;      // candidates = B n_cand
    int B = 0;
};

uh_status check_common(int32_t K, const uh_mot_branch* br, int32_t n_cand, int32_t d, uh_dtype dt, MotShape* s) {
    if (!br) return fail(UH_ERR_NULL, "branches is NULL");
    if (K < 1 || n_cand < 1 || d < 1) return fail(UH_ERR_DOMAIN, "n_branches, n_cand and d must be >= 1");
    if (K > kMaxBranches) return fail(UH_ERR_UNSUPPORTED, "at most 8 branches");
    if (dt != UH_BF16 && dt != UH_F32) return fail(UH_ERR_DOMAIN, "unknown dtype");
    if (dt == UH_BF16 && d % 64) return fail(UH_ERR_SHAPE, "bf16 MoT fusion needs d % 64 == 0");
    const int es = dt == UH_BF16 ? 2 : 4;
    if (((int64_t)d * es) % 16) return fail(UH_ERR_ALIGNMENT, "d * element size must be a multiple of 16 bytes");
    for (int k = 0; k < K; ++k) {
        UH_TRY(validate_jagged(br[k].jag, true));
        if (br[k].jag->num_seqs != br[0].jag->num_seqs)
            return fail(UH_ERR_DIM, "branches hold different user counts (R29)");
        if (!br[k].x && br[k].jag->total_tokens > 0) return fail(UH_ERR_NULL, "branch x is NULL");
        if (!aligned16(br[k].x) || br[k].ld < d || (br[k].ld * es) % 16)
            return fail(UH_ERR_ALIGNMENT, "branch x must be 16-byte aligned with ld >= d, ld * elem % 16 == 0");
        const int32_t* o = br[k].jag->host_offsets;
        for (int b = 0; b < br[k].jag->num_seqs; ++b)
            if (o[b + 1] - o[b] < n_cand)
                return fail(UH_ERR_DIM, "branch " + std::to_string(k) + " sequence " + std::to_string(b) +
                                            " is shorter than n_cand (R29)");
    }
    s->B = br[0].jag->num_seqs;
    s->C = (int64_t)s->B * n_cand;
    if (s->C * K * (int64_t)d > INT32_MAX) return fail(UH_ERR_UNSUPPORTED, "C * K * d exceeds 2^31-1");
    return UH_OK;
}

MotRows rows_of(int32_t K, const uh_mot_branch* br, void* const* dx, const int64_t* ld_dx, int es) {
    MotRows r{};
    r.n = K;
    for (int k = 0; k < K; ++k) {
        r.x[k] = dx ? static_cast<uint8_t*>(dx[k]) : static_cast<uint8_t*>(const_cast<void*>(br[k].x));
        r.ld_bytes[k] = (dx ? ld_dx[k] : br[k].ld) * es;
        r.off[k] = br[k].jag->offsets;
    }
    return r;
}

template <bool SCATTER>
uh_status launch_rows(const MotRows& r, int64_t C, int n_cand, int64_t row_bytes, void* z, int64_t ldz_bytes,
                      cudaStream_t st) {
    const int64_t warps = C * r.n;
    if (warps == 0) return UH_OK;
    const int blocks = (int)std::min<int64_t>((warps + 7) / 8, 8LL * num_sms());
    mot_rows_k<SCATTER><<<blocks, 256, 0, st>>>(r, C, n_cand, row_bytes, static_cast<uint8_t*>(z), ldz_bytes);
    note_launch();
    UH_CUDA(cudaGetLastError());
    return UH_OK;
}

}  // namespace
}  // namespace uh

using namespace uh;

extern "C" uh_status uh_mot_workspace_bytes(int32_t K, const uh_mot_branch* br, int32_t n_cand, int32_t d,
                                            uh_dtype dt, int backward, size_t* bytes) {
    if (!bytes) return fail(UH_ERR_NULL, "bytes is NULL");
    MotShape s;
    UH_TRY(check_common(K, br, n_cand, d, dt, &s));
    const size_t z = round256((size_t)s.C * K * d * (dt == UH_BF16 ? 2 : 4));
    *bytes = backward ? 2 * z : z;
    return UH_OK;
}

extern "C" uh_status uh_mot_fuse_fwd(int32_t K, const uh_mot_branch* br, int32_t n_cand, int32_t d, uh_dtype dt,
                                     const void* w_f, const float* b_f, void* e, void* ws, size_t ws_bytes,
                                     void* stream) {
    MotShape s;
    UH_TRY(check_common(K, br, n_cand, d, dt, &s));
    if (s.C == 0) return UH_OK;
    if (!w_f || !e) return fail(UH_ERR_NULL, "w_f / e is NULL");
    if (!aligned16(w_f) || !aligned16(e) || !aligned16(b_f)) return fail(UH_ERR_ALIGNMENT, "w_f, b_f, e 16-byte aligned");
    const int es = dt == UH_BF16 ? 2 : 4;
    const size_t zb = round256((size_t)s.C * K * d * es);
    if (!ws || ws_bytes < zb) return fail(UH_ERR_WORKSPACE, "workspace too small: need " + std::to_string(zb));
    if (!aligned16(ws)) return fail(UH_ERR_ALIGNMENT, "workspace 16-byte aligned");
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t ldz = (int64_t)K * d;
    UH_TRY(launch_rows<false>(rows_of(K, br, nullptr, nullptr, es), s.C, n_cand, (int64_t)d * es, ws, ldz * es, st));
    GemmDesc g;                      // E = Z W_f + b_f: A = Z [C][K d], B = W_f [K d][d] (MN-major)
    g.M = (int)s.C; g.N = d; g.K = K * d;
    g.A = ws; g.lda = ldz; g.a_mn = false;
    g.B = w_f; g.ldb = d; g.b_mn = true;
    g.epi = EPI_BF16; g.out0 = e; g.ld0 = d; g.bias = b_f;
    return gemm_run(g, dt, st);
}

extern "C" uh_status uh_mot_fuse_bwd(int32_t K, const uh_mot_branch* br, int32_t n_cand, int32_t d, uh_dtype dt,
                                     const void* w_f, const void* de, float* dw_f, float* db_f, int accumulate,
                                     void* const* dx, const int64_t* ld_dx, void* ws, size_t ws_bytes,
                                     void* stream) {
    MotShape s;
    UH_TRY(check_common(K, br, n_cand, d, dt, &s));
    if (!w_f || !de || !dw_f || !dx || !ld_dx) return fail(UH_ERR_NULL, "w_f / de / dw_f / dx / ld_dx is NULL");
    const int es = dt == UH_BF16 ? 2 : 4;
    for (int k = 0; k < K; ++k) {
        if (!dx[k] && br[k].jag->total_tokens > 0) return fail(UH_ERR_NULL, "dx[k] is NULL");
        if (!aligned16(dx[k]) || ld_dx[k] < d || (ld_dx[k] * es) % 16)
            return fail(UH_ERR_ALIGNMENT, "dx[k] 16-byte aligned with ld_dx >= d, ld_dx * elem % 16 == 0");
    }
    if (!aligned16(w_f) || !aligned16(de) || !aligned16(dw_f) || !aligned16(db_f))
        return fail(UH_ERR_ALIGNMENT, "w_f, de, dw_f, db_f 16-byte aligned");
    const size_t zb = round256((size_t)s.C * K * d * es);
    if (s.C > 0 && (!ws || ws_bytes < 2 * zb))
        return fail(UH_ERR_WORKSPACE, "workspace too small: need " + std::to_string(2 * zb));
    if (!aligned16(ws)) return fail(UH_ERR_ALIGNMENT, "workspace 16-byte aligned");
    cudaStream_t st = (cudaStream_t)stream;
    if (!accumulate) {
        UH_CUDA(cudaMemsetAsync(dw_f, 0, (size_t)K * d * d * sizeof(float), st));
        if (db_f) UH_CUDA(cudaMemsetAsync(db_f, 0, (size_t)d * sizeof(float), st));
    }
    for (int k = 0; k < K; ++k)      // every row of dX_k outside the candidates is zero (R30)
        if (br[k].jag->total_tokens > 0)
            UH_CUDA(cudaMemset2DAsync(dx[k], (size_t)ld_dx[k] * es, 0, (size_t)d * es, (size_t)br[k].jag->total_tokens, st));
    if (s.C == 0) return UH_OK;
    uint8_t* Z = static_cast<uint8_t*>(ws);
    uint8_t* dZ = Z + zb;
    const int64_t ldz = (int64_t)K * d;
    UH_TRY(launch_rows<false>(rows_of(K, br, nullptr, nullptr, es), s.C, n_cand, (int64_t)d * es, Z, ldz * es, st));
    GemmDesc gz;                     // dZ = dE W_f^T: B = W_f^T, i.e. W_f [K d][d] read as [N][K] (K-major)
    gz.M = (int)s.C; gz.N = K * d; gz.K = d;
    gz.A = de; gz.lda = d; gz.a_mn = false;
    gz.B = w_f; gz.ldb = d; gz.b_mn = false;
    gz.epi = EPI_BF16; gz.out0 = dZ; gz.ld0 = ldz;
    UH_TRY(gemm_run(gz, dt, st));
    UH_TRY(launch_rows<true>(rows_of(K, br, dx, ld_dx, es), s.C, n_cand, (int64_t)d * es, dZ, ldz * es, st));
    GemmDesc gw;                     // dW_f = Z^T dE: A = Z^T ([C][K d] = [K][M], MN-major), B = dE ([K][N])
    gw.M = K * d; gw.N = d; gw.K = (int)s.C;
    gw.A = Z; gw.lda = ldz; gw.a_mn = true;
    gw.B = de; gw.ldb = d; gw.b_mn = true;
    gw.epi = EPI_F32; gw.out0 = dw_f; gw.ld0 = d;
    const bool fuse_cs = dt == UH_BF16 && d % 256 == 0 && (K * d) % 256 == 0;
    if (db_f && fuse_cs) gw.colsum = db_f;
    UH_TRY(gemm_run(gw, dt, st));
    if (db_f && !fuse_cs) UH_TRY(colsum(dt, s.C, d, de, d, db_f, st));
    return UH_OK;
}
