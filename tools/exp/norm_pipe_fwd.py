# norms: the forward row kernels (LN, LN from saved statistics, gated norm) stream their rows through
# the per-warp bulk-copy rings the backward row kernels already use (4 rows in flight per warp,
# persistent grid), instead of one warp per row with two 16-byte loads in flight per lane
KERNEL = r'''
// MODE 0: y = LN(x) (stats out); 1: y = LN(x) from saved stats; 2: y = LN(x) (.) u (stats out)
template <int CPL, int DEPTH, int MODE>
__global__ void __launch_bounds__(256) norm_fwd_pipe_k(int64_t nrows, int d, const __nv_bfloat16* __restrict__ x,
                                                      int64_t ldx, const __nv_bfloat16* __restrict__ u, int64_t ldu,
                                                      const float* __restrict__ w, const float* __restrict__ b,
                                                      float eps, __nv_bfloat16* __restrict__ y, int64_t ldy,
                                                      float* mean, float* rstd) {
    using T = __nv_bfloat16;
    constexpr int V = 8, NT = MODE == 2 ? 2 : 1;
    extern __shared__ __align__(128) uint8_t pipe_smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int rb = d * 2, nch = d / V;
    uint64_t* bars = reinterpret_cast<uint64_t*>(pipe_smem + 2 * d * 4);
    uint8_t* ring0 = pipe_smem + 2 * d * 4 + kPipeWarps * DEPTH * 8;
    ring0 += (128 - (reinterpret_cast<uintptr_t>(ring0) & 127)) & 127;
    RowRing<NT, DEPTH> rr{ring0 + (size_t)warp * DEPTH * NT * rb, bars + warp * DEPTH, rb};
    const uint8_t* src[2] = {reinterpret_cast<const uint8_t*>(x), reinterpret_cast<const uint8_t*>(u)};
    const int64_t ldb[2] = {ldx * 2, ldu * 2};
    const int64_t G = (int64_t)gridDim.x * kPipeWarps;
    const int64_t r0 = (int64_t)blockIdx.x * kPipeWarps + warp;
    if (lane == 0) {
        for (int s = 0; s < DEPTH; ++s) mbar_init(&rr.bar[s], 1);
        fence_barrier_init();
        for (int s = 0; s < DEPTH; ++s)
            if (r0 + s * G < nrows) rr.issue(s, src, ldb, r0 + s * G);
    }
    __syncwarp();
    float wv[CPL][V], bv[CPL][V];
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
        const int ch = lane + 32 * c;
#pragma unroll
        for (int e = 0; e < V; ++e) { wv[c][e] = 0.f; bv[c][e] = 0.f; }
        if (ch < nch)
#pragma unroll
            for (int e = 0; e < V; e += 4) { load4f(w + ch * V + e, wv[c] + e); load4f(b + ch * V + e, bv[c] + e); }
    }
    float mu_n = 0.f, rs_n = 0.f;
    if (MODE == 1 && r0 < nrows) { mu_n = mean[r0]; rs_n = rstd[r0]; }
    int k = 0;
    for (int64_t row = r0; row < nrows; row += G, ++k) {
        const int s = k % DEPTH;
        float mu = mu_n, rs = rs_n;
        if (MODE == 1 && row + G < nrows) { mu_n = mean[row + G]; rs_n = rstd[row + G]; }
        mbar_wait(&rr.bar[s], (k / DEPTH) & 1);
        float xv[CPL][V], uv[CPL][V];
        float sum = 0.f;
#pragma unroll
        for (int c = 0; c < CPL; ++c) {
            const int ch = lane + 32 * c;
            if (ch < nch) {
                bf16x8_to_f32(*reinterpret_cast<const uint4*>(rr.slot(s, 0) + ch * 16), xv[c]);
                if (MODE == 2) bf16x8_to_f32(*reinterpret_cast<const uint4*>(rr.slot(s, 1) + ch * 16), uv[c]);
#pragma unroll
                for (int e = 0; e < V; ++e) sum += xv[c][e];
            }
        }
        __syncwarp();
        if (lane == 0 && row + DEPTH * G < nrows) rr.issue(s, src, ldb, row + DEPTH * G);
        if (MODE != 1) {
            mu = warp_sum(sum) / d;
            float q = 0.f;
#pragma unroll
            for (int c = 0; c < CPL; ++c)
                if (lane + 32 * c < nch)
#pragma unroll
                    for (int e = 0; e < V; ++e) { const float t = xv[c][e] - mu; q += t * t; }
            rs = rsqrtf(warp_sum(q) / d + eps);
        }
#pragma unroll
        for (int c = 0; c < CPL; ++c) {
            const int ch = lane + 32 * c;
            if (ch < nch) {
                float o[V];
#pragma unroll
                for (int e = 0; e < V; ++e) {
                    o[e] = (xv[c][e] - mu) * rs * wv[c][e] + bv[c][e];
                    if (MODE == 2) o[e] *= uv[c][e];
                }
                Vec<T>::store(y + row * ldy + ch * V, o);
            }
        }
        if (MODE != 1 && lane == 0) {
            if (mean) mean[row] = mu;
            if (rstd) rstd[row] = rs;
        }
    }
}

'''
HOOK = "// ------------------------------------------------------------------ column sums / scale"
LNF_OLD = """    if (T_ == 0) return UH_OK;
    UH_DT_DISPATCH(dt, UH_CPL_DISPATCH(T, d,
        ln_fwd_k<T, CPL><<<grid_rows(T_), 256, 0, st>>>(T_, d, (const T*)x, ldx, w, b, eps, (T*)y, ldy, mean, rstd)));"""
LNF_NEW = """    if (T_ == 0) return UH_OK;
    if (dt == UH_BF16 && pipe_ok(d, {{x, ldx}, {y, ldy}})) {
        using T = __nv_bfloat16;
        const size_t sm = pipe_smem_bytes<1>(d);
        const int blocks = (int)std::min<int64_t>(2LL * num_sms(), (T_ + kPipeWarps - 1) / kPipeWarps);
        UH_PIPE_CPL(d, {
            UH_CUDA(cudaFuncSetAttribute(norm_fwd_pipe_k<CPL, kPipeDepth, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
            norm_fwd_pipe_k<CPL, kPipeDepth, 0><<<blocks, 256, sm, st>>>(T_, d, (const T*)x, ldx, nullptr, 0, w, b, eps,
                                                                         (T*)y, ldy, mean, rstd);
        });
        note_launch();
        UH_CUDA(cudaGetLastError());
        return UH_OK;
    }
    UH_DT_DISPATCH(dt, UH_CPL_DISPATCH(T, d,
        ln_fwd_k<T, CPL><<<grid_rows(T_), 256, 0, st>>>(T_, d, (const T*)x, ldx, w, b, eps, (T*)y, ldy, mean, rstd)));"""
LNA_OLD = """    if (T_ == 0) return UH_OK;
    UH_DT_DISPATCH(dt, UH_CPL_DISPATCH(T, d,
        ln_apply_k<T, CPL><<<grid_rows(T_), 256, 0, st>>>(T_, d, (const T*)x, ldx, w, b, mean, rstd, (T*)y, ldy)));"""
LNA_NEW = """    if (T_ == 0) return UH_OK;
    if (dt == UH_BF16 && pipe_ok(d, {{x, ldx}, {y, ldy}})) {
        using T = __nv_bfloat16;
        const size_t sm = pipe_smem_bytes<1>(d);
        const int blocks = (int)std::min<int64_t>(2LL * num_sms(), (T_ + kPipeWarps - 1) / kPipeWarps);
        UH_PIPE_CPL(d, {
            UH_CUDA(cudaFuncSetAttribute(norm_fwd_pipe_k<CPL, kPipeDepth, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
            norm_fwd_pipe_k<CPL, kPipeDepth, 1><<<blocks, 256, sm, st>>>(T_, d, (const T*)x, ldx, nullptr, 0, w, b, 0.f,
                                                                         (T*)y, ldy, const_cast<float*>(mean),
                                                                         const_cast<float*>(rstd));
        });
        note_launch();
        UH_CUDA(cudaGetLastError());
        return UH_OK;
    }
    UH_DT_DISPATCH(dt, UH_CPL_DISPATCH(T, d,
        ln_apply_k<T, CPL><<<grid_rows(T_), 256, 0, st>>>(T_, d, (const T*)x, ldx, w, b, mean, rstd, (T*)y, ldy)));"""
GF_OLD = """    if (T_ == 0) return UH_OK;
    UH_DT_DISPATCH(dt, UH_CPL_DISPATCH(T, d,
        gated_fwd_k<T, CPL><<<grid_rows(T_), 256, 0, st>>>(T_, d, (const T*)A, lda, (const T*)U, ldu, w, b, eps,
                                                           (T*)Y, ldy, mean, rstd)));"""
GF_NEW = """    if (T_ == 0) return UH_OK;
    if (dt == UH_BF16 && pipe_ok(d, {{A, lda}, {U, ldu}, {Y, ldy}})) {
        using T = __nv_bfloat16;
        const size_t sm = pipe_smem_bytes<2>(d);
        const int blocks = (int)std::min<int64_t>(2LL * num_sms(), (T_ + kPipeWarps - 1) / kPipeWarps);
        UH_PIPE_CPL(d, {
            UH_CUDA(cudaFuncSetAttribute(norm_fwd_pipe_k<CPL, kPipeDepth, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
            norm_fwd_pipe_k<CPL, kPipeDepth, 2><<<blocks, 256, sm, st>>>(T_, d, (const T*)A, lda, (const T*)U, ldu, w, b,
                                                                         eps, (T*)Y, ldy, mean, rstd);
        });
        note_launch();
        UH_CUDA(cudaGetLastError());
        return UH_OK;
    }
    UH_DT_DISPATCH(dt, UH_CPL_DISPATCH(T, d,
        gated_fwd_k<T, CPL><<<grid_rows(T_), 256, 0, st>>>(T_, d, (const T*)A, lda, (const T*)U, ldu, w, b, eps,
                                                           (T*)Y, ldy, mean, rstd)));"""
PATCHES = [("norm.cu", HOOK, KERNEL + HOOK), ("norm.cu", LNF_OLD, LNF_NEW), ("norm.cu", LNA_OLD, LNA_NEW),
           ("norm.cu", GF_OLD, GF_NEW)]
