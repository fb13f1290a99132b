# bwd P/dS warps: take the next work item (and prefetch its key-row / first-step timestamps into
# L1) before the current item's acc_full wait, which hides those dependent global loads
OLD1 = """        int sc = 0, ki = 0;
        for (;; ++ki) {
            const int w = ring_take(&bars->ring, ki, lane);
            if (w < 0) break;
            const WorkItem it = a.items[w];
            check_item(a, it, BM);
            const int L = it.seq_len, o = it.seq_start, h = it.head & 0xFFFF;
            const int k0 = it.tile * BM;
            const int n = n_qtiles(k0, L, a.K1, a.K2);
            const int kp = k0 + r;"""
NEW1 = """        int sc = 0, ki = 0;
        int w = ring_take(&bars->ring, 0, lane);
        WorkItem itn{};
        if (w >= 0) itn = a.items[w];
        for (;; ++ki) {
            if (w < 0) break;
            const WorkItem it = itn;
            check_item(a, it, BM);
            const int L = it.seq_len, o = it.seq_start, h = it.head & 0xFFFF;
            const int k0 = it.tile * BM;
            const int n = n_qtiles(k0, L, a.K1, a.K2);
            const int kp = k0 + r;"""
OLD2 = """            if (run_v != 0.f) atomicAdd(dts_l + run_b * DTS_LANES, run_v);
            mbar_wait_sleep(&bars->acc_full, ki & 1);"""
NEW2 = """            if (run_v != 0.f) atomicAdd(dts_l + run_b * DTS_LANES, run_v);
            {   // the next item before this one's acc_full wait (which hides its loads)
                const int wn = ring_take(&bars->ring, ki + 1, lane);
                if (wn >= 0) {
                    itn = a.items[wn];
                    if (a.ts) {
                        const int64_t* tp = a.t + itn.seq_start;
                        const int kn = itn.tile * BM, qbn = (kn / BN) * BN + 32 * wg;
                        asm volatile("prefetch.global.L1 [%0];" ::"l"(tp));
                        asm volatile("prefetch.global.L1 [%0];" ::"l"(tp + imin(kn + r, itn.seq_len - 1)));
                        asm volatile("prefetch.global.L1 [%0];" ::"l"(tp + imin(qbn + lane, itn.seq_len - 1)));
                    }
                }
                w = wn;
            }
            mbar_wait_sleep(&bars->acc_full, ki & 1);"""
PATCHES = [("attn_bwd_sm100.cu", OLD1, NEW1), ("attn_bwd_sm100.cu", OLD2, NEW2)]
