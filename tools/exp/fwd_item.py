# fwd epilogue: the next work item is taken (and its WorkItem, row / first-tile timestamps
# prefetched into L1) before the current item's O epilogue, whose o_full wait hides the
# dependent global loads that otherwise stall every warpgroup at each item start
OLD1 = """        int sc = 0, qi = 0;
        for (;; ++qi) {
            const int w = ring_take(&bars->ring, qi, lane);
            if (w < 0) break;
            const WorkItem it = a.items[w];"""
NEW1 = """        int sc = 0, qi = 0;
        int w = ring_take(&bars->ring, 0, lane);
        WorkItem itn{};
        if (w >= 0) itn = a.items[w];
        for (;; ++qi) {
            if (w < 0) break;
            const WorkItem it = itn;"""
OLD2 = """            // ---- O epilogue: A = O / N (32 columns per warpgroup)
            mbar_wait_sleep(&bars->o_full, qi & 1);"""
NEW2 = """            // the next item before this one's O epilogue (the o_full wait hides its loads)
            const int wn = ring_take(&bars->ring, qi + 1, lane);
            if (wn >= 0) {
                itn = a.items[wn];
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
            mbar_wait_sleep(&bars->o_full, qi & 1);"""
PATCHES = [("attn_fwd_sm100.cu", OLD1, NEW1), ("attn_fwd_sm100.cu", OLD2, NEW2)]
