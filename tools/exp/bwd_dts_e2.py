# bwd: the d time_bias runs move from the P/dS warps (the step's critical path) to the dQ warps,
# which have slack and already load each row's 32 bf16 dS' values for d pos_bias: same thread ->
# (key row, 32 query columns) map, same chunk classification (recomputed), bf16 instead of fp32
# dS' terms (R15b bound).  Registers: P/dS 136 -> 128, dQ 80 -> 88.
E1_DTS_OLD = """                if (a.dts) {   // runs of equal time bucket along the row (FLAG_T1: two, FLAG_T2: per element)
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
            if (run_v != 0.f) atomicAdd(dts_l + run_b * DTS_LANES, run_v);"""
E1_DTS_NEW = """            }"""
E1_FLUSH_OLD = """        // the CTA's d time_bias partials -> one global atomic per bucket
        __syncwarp();
        named_bar_sync(4, 256);
        const int t = threadIdx.x - 128;
        if (a.dts && t < a.NB) {
            float v = 0.f;
#pragma unroll
            for (int l = 0; l < DTS_LANES; ++l) v += dts_s[t * DTS_LANES + l];
            if (v != 0.f) atomicAdd(a.dts + t, v * (0.5f * a.inv_n));
        }
    } else {"""
E1_FLUSH_NEW = """    } else {"""
E2_ITEM_OLD = """            const int k0 = it.tile * BM;
            const int n = n_qtiles(k0, L, a.K1, a.K2);
            for (int i = 0; i < n; ++i, ++sc) {
                const int sb = sc & 1;
                const int qb0 = (k0 / BN + i) * BN;
                mbar_wait_sleep(&bars->dq_full[sb], (sc >> 1) & 1);"""
E2_ITEM_NEW = """            const int k0 = it.tile * BM;
            const int n = n_qtiles(k0, L, a.K1, a.K2);
            // d time_bias runs of this thread's key row (as the P/dS warps' rows)
            const int kp = k0 + r;
            const bool kok = kp < L;
            const ChunkCtx cx = make_ctx(a, ts_s, o, L);
            const int32_t tk = (a.ts && kok) ? rel32(__ldg(a.t + o + kp), cx.t0) : 0;
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
                const int qb0 = (k0 / BN + i) * BN;
                mbar_wait_sleep(&bars->dq_full[sb], (sc >> 1) & 1);"""
E2_POS_OLD = """                if (a.dpos) {
                    // d pos_bias[min(q - k, P - 1)] += ds: in this warp's 32 x 32 block of dS^T the
                    // element (row s, column c) sits on diagonal C + c - s; a skewed shuffle (lane m
                    // reads column c from lane (c - m) mod 32) gives lane m the sums of diagonals
                    // C + m (c >= m) and C + m - 32 (c < m): two global reductions per lane and
                    // block; blocks whose offsets all clamp to P - 1 accumulate in a register.
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
                        if (C - 31 >= a.P - 1) {"""
E2_POS_NEW = """                uint32_t d2[16];
                const int C = qb0 + 32 * hf - k0 - 32 * wq;
                const bool have = (a.dpos || a.dts) && C + 31 >= 0;   // warp-uniform: else strictly upper (masked)
                if (have) {
                    mbar_wait(&bars->p_full[sb], (sc >> 1) & 1);   // the P/dS warps' shared stores are visible
                    const uint8_t* row = sDS + sb * DS_BYTES + r * 128;
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        const uint4 u = *reinterpret_cast<const uint4*>(row + (((4 * hf + c) ^ (r & 7)) << 4));
                        d2[4 * c] = u.x; d2[4 * c + 1] = u.y; d2[4 * c + 2] = u.z; d2[4 * c + 3] = u.w;
                    }
                }
                if (a.dpos) {
                    // d pos_bias[min(q - k, P - 1)] += ds: in this warp's 32 x 32 block of dS^T the
                    // element (row s, column c) sits on diagonal C + c - s; a skewed shuffle (lane m
                    // reads column c from lane (c - m) mod 32) gives lane m the sums of diagonals
                    // C + m (c >= m) and C + m - 32 (c < m): two global reductions per lane and
                    // block; blocks whose offsets all clamp to P - 1 accumulate in a register.
                    if (have) {
                        if (C - 31 >= a.P - 1) {"""
E2_FREE_OLD = """                __syncwarp();
                if (lane == 0) mbar_arrive(&bars->ds_free[sb]);
                if (warp == 12) TRACE_FB(6, sc);
            }
        }"""
E2_FREE_NEW = """                __syncwarp();
                if (lane == 0) mbar_arrive(&bars->ds_free[sb]);
                if (warp == 12) TRACE_FB(6, sc);
                if (a.dts && have) {   // runs of equal time bucket along the row (FLAG_T1: two, FLAG_T2: per element)
                    const int qb = qb0 + 32 * hf;
                    const Chunk ch = k_chunk(cx, kp, kok, tk, qb, col_time(cx, qb, lane));
                    float dp[32];
#pragma unroll
                    for (int c = 0; c < 16; ++c) {
                        const float2 u = unpack_bf16x2(d2[c]);
                        dp[2 * c] = u.x; dp[2 * c + 1] = u.y;
                    }
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
        }
        // the CTA's d time_bias partials -> one global atomic per bucket
        __syncwarp();
        named_bar_sync(4, 256);
        {
            const int t = threadIdx.x - 384;
            if (a.dts && t < a.NB) {
                float v = 0.f;
#pragma unroll
                for (int l = 0; l < DTS_LANES; ++l) v += dts_s[t * DTS_LANES + l];
                if (v != 0.f) atomicAdd(a.dts + t, v * (0.5f * a.inv_n));
            }
        }"""
PATCHES = [
    ("attn_bwd_sm100.cu", E1_DTS_OLD, E1_DTS_NEW),
    ("attn_bwd_sm100.cu", E1_FLUSH_OLD, E1_FLUSH_NEW),
    ("attn_bwd_sm100.cu", E2_ITEM_OLD, E2_ITEM_NEW),
    ("attn_bwd_sm100.cu", E2_POS_OLD, E2_POS_NEW),
    ("attn_bwd_sm100.cu", E2_FREE_OLD, E2_FREE_NEW),
    ("attn_bwd_sm100.cu", "constexpr int REG_LAUNCH = 96, REG_CTRL = 48, REG_PDS = 136, REG_DQ = 80;",
     "constexpr int REG_LAUNCH = 96, REG_CTRL = 48, REG_PDS = 128, REG_DQ = 88;"),
]
