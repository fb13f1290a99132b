# bwd E1: software-pipelined rab — the next step's chunk classification and position-table pair
# loads are issued before the current step's d time_bias work (timestamps two steps ahead), and the
# bias is formed before the S wait; after the TMEM load only h = alpha/2 S + bias remains.
HELPERS = r'''
// ---- key-row (backward) rab in two phases, for software pipelining across query steps:
// k_pos_issue loads the chunk's 16 position-table pairs (FLAG_P), k_bias forms the bias of
// h = alpha/2 S + bias from them (T1 bucket split, T2 per-element buckets included).
UH_DEV void k_pos_issue(const ChunkCtx& c, const Chunk& ch, float2* pe) {
    if (ch.flags & FLAG_P) {
        const int i0 = ch.bd + kPosOff;
        UH_CHECK(i0 >= 0 && i0 + 33 < c.Lt);
        const float* p = c.pe - kPosOff + (i0 & 1) * c.Lt + (i0 & ~1);
#pragma unroll
        for (int j = 0; j < 16; ++j) pe[j] = pe_pair(p + 2 * j);
    }
}
UH_DEV void k_bias(const ChunkCtx& c, const Chunk& ch, int32_t tk, const float2* pe, float* b) {
    const float hb = ch.hbias, ho = ch.hbias_o;
    const bool t1 = ch.flags & FLAG_T1, p = ch.flags & FLAG_P;
#pragma unroll
    for (int j = 0; j < 32; j += 2) {
        float b0 = hb, b1 = hb;
        if (t1) {
            b0 = j >= ch.n ? ho : hb;
            b1 = j + 1 >= ch.n ? ho : hb;
        }
        if (p) {
            b0 += pe[j >> 1].x;
            b1 += pe[j >> 1].y;
        }
        b[j] = b0; b[j + 1] = b1;
    }
    if (ch.flags & FLAG_T2) {
        const float tb = c.ts_h[ch.b_base];
        const bool multi = !(ch.b_other == ch.b_base + 1 || ch.b_other == ch.b_base);
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            const int32_t tc = __shfl_sync(0xffffffffu, ch.tcol, j);
            b[j] += multi ? c.ts_h[bucket32(tc - tk, c.NB)] - tb : 0.f;
        }
    }
}
'''
OLD_TOP = """            for (int i = 0; i < n; ++i, ++sc) {
                const int sb = sc & 1;
                const int qb = (k0 / BN + i) * BN + 32 * wg;   // this warpgroup's 32 queries
                const int32_t tcur = col_time(cx, qb, lane);
                const Chunk ch = k_chunk(cx, kp, kok, tk, qb, tcur);
                mbar_wait_sleep(&bars->s_full[sb], (sc >> 1) & 1);"""
NEW_TOP = """            // software pipeline over the query steps: step i's chunk and position pairs were
            // prepared during step i-1 (timestamps two steps ahead), its bias before the S wait
            const int qb0 = (k0 / BN) * BN + 32 * wg;
            Chunk ch = k_chunk(cx, kp, kok, tk, qb0, col_time(cx, qb0, lane));
            int32_t t_nxt = n > 1 ? col_time(cx, qb0 + BN, lane) : 0;
            float2 pe2[16];
            k_pos_issue(cx, ch, pe2);
            for (int i = 0; i < n; ++i, ++sc) {
                const int sb = sc & 1;
                const int qb = (k0 / BN + i) * BN + 32 * wg;   // this warpgroup's 32 queries
                float hx[32];
                k_bias(cx, ch, tk, pe2, hx);
                mbar_wait_sleep(&bars->s_full[sb], (sc >> 1) & 1);"""
OLD_H = """                float hx[32];
                k_h(cx, ch, tk, sv, hx);"""
NEW_H = """                {
                    const uint64_t A2 = f2_pack(cx.ha, cx.ha);
#pragma unroll
                    for (int j = 0; j < 32; j += 2) {
                        const float2 v = f2_unpack(ffma2(f2_pack(sv[j], sv[j + 1]), A2, f2_pack(hx[j], hx[j + 1])));
                        hx[j] = v.x; hx[j + 1] = v.y;
                    }
                }"""
OLD_DTS = """                if (warp == 4) TRACE_FB(3, sc);
                if (a.dts) {"""
NEW_DTS = """                if (warp == 4) TRACE_FB(3, sc);
                const Chunk chc = ch;
                if (i + 1 < n) {   // next step: classify (its timestamps were loaded a step ago), issue its pairs
                    ch = k_chunk(cx, kp, kok, tk, qb + BN, t_nxt);
                    t_nxt = i + 2 < n ? col_time(cx, qb + 2 * BN, lane) : 0;
                    k_pos_issue(cx, ch, pe2);
                }
                if (a.dts) {"""
PATCHES = [
    ("attn_common.cuh", "// query-row chunk (forward)", HELPERS + "\n// query-row chunk (forward)"),
    ("attn_bwd_sm100.cu", OLD_TOP, NEW_TOP),
    ("attn_bwd_sm100.cu", OLD_H, NEW_H),
    ("attn_bwd_sm100.cu", OLD_DTS, NEW_DTS),
]
OLD_DTSB = """                    if (!(ch.flags & FLAG_T2)) {
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
                    }"""
PATCHES.append(("attn_bwd_sm100.cu", OLD_DTSB, OLD_DTSB.replace("ch.", "chc.")))
