# fwd epilogue: the next item's row timestamps (t0, tq) are loaded into registers before the O
# epilogue's row stores (which otherwise queue ahead of them in the LSU), and pos[P-1] once per CTA
OLD0 = """        int sc = 0, qi = 0;
        int w = ring_take(&bars->ring, 0, lane);
        WorkItem itn{};
        if (w >= 0) itn = a.items[w];"""
NEW0 = """        int sc = 0, qi = 0;
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
        const float pos_far = a.pos ? 0.5f * __ldg(a.pos + a.P - 1) : 0.f;"""
OLD1 = """            const ChunkCtx cx = make_ctx(a, ts_s, o, L);
            const int32_t tq = (a.ts && qok) ? rel32(__ldg(a.t + o + qp), cx.t0) : 0;
            // tiles rotate over the four warpgroups"""
NEW1 = """            ChunkCtx cx;
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
            // tiles rotate over the four warpgroups"""
OLD2 = """            if (wn >= 0) {
                itn = a.items[wn];
                if (a.ts) {"""
NEW2 = """            if (wn >= 0) {
                itn = a.items[wn];
                load_rowtimes(itn);
                if (a.ts) {"""
PATCHES = [("attn_fwd_sm100.cu", OLD0, NEW0), ("attn_fwd_sm100.cu", OLD1, NEW1), ("attn_fwd_sm100.cu", OLD2, NEW2)]
