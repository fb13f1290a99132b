# fwd (4 warpgroups): each warpgroup prefetches the column timestamps of its next tile (j + 4)
OLD = """            for (int j = 0; j < n; ++j, ++sc) {
                if ((sc & 3) != wg) continue;
                const int sb = sc % NS;
                const int k0 = key_tile_at(kt, j) * BN;
                const int32_t tc0 = col_time(cx, k0, lane), tc1 = col_time(cx, k0 + 32, lane);"""
NEW = """            int32_t pf0 = 0, pf1 = 0;
            int pf_j = -1;
            for (int j = 0; j < n; ++j, ++sc) {
                if ((sc & 3) != wg) continue;
                const int sb = sc % NS;
                const int k0 = key_tile_at(kt, j) * BN;
                int32_t tc0 = pf0, tc1 = pf1;
                if (pf_j != j) { tc0 = col_time(cx, k0, lane); tc1 = col_time(cx, k0 + 32, lane); }
                if (j + 4 < n) {   // this warpgroup's next tile of the item: its timestamps a tile ahead
                    const int kn = key_tile_at(kt, j + 4) * BN;
                    pf0 = col_time(cx, kn, lane); pf1 = col_time(cx, kn + 32, lane); pf_j = j + 4;
                }"""
PATCHES = [("attn_fwd_sm100.cu", OLD, NEW)]
