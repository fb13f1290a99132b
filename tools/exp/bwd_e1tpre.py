# bwd E1: only the column timestamps are prefetched one query step ahead (no other pipelining)
OLD = """            for (int i = 0; i < n; ++i, ++sc) {
                const int sb = sc & 1;
                const int qb = (k0 / BN + i) * BN + 32 * wg;   // this warpgroup's 32 queries
                const int32_t tcur = col_time(cx, qb, lane);
                const Chunk ch = k_chunk(cx, kp, kok, tk, qb, tcur);"""
NEW = """            int32_t t_nxt = col_time(cx, (k0 / BN) * BN + 32 * wg, lane);
            for (int i = 0; i < n; ++i, ++sc) {
                const int sb = sc & 1;
                const int qb = (k0 / BN + i) * BN + 32 * wg;   // this warpgroup's 32 queries
                const int32_t tcur = t_nxt;
                if (i + 1 < n) t_nxt = col_time(cx, qb + BN, lane);   // next step's, a step ahead
                const Chunk ch = k_chunk(cx, kp, kok, tk, qb, tcur);"""
PATCHES = [("attn_bwd_sm100.cu", OLD, NEW)]
