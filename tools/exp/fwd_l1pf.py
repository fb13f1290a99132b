# fwd epilogue: prefetch.global.L1 of the warpgroup's next tile's (j + 4) column timestamps and
# position-table pairs (no registers held)
OLD = """                const int32_t tc0 = col_time(cx, k0, lane), tc1 = col_time(cx, k0 + 32, lane);"""
NEW = """                const int32_t tc0 = col_time(cx, k0, lane), tc1 = col_time(cx, k0 + 32, lane);
                if (j + 4 < n) {   // this warpgroup's next tile: timestamps and position pairs into L1
                    const int kn = key_tile_at(kt, j + 4) * BN;
                    if (cx.ts_h) {
                        asm volatile("prefetch.global.L1 [%0];" ::"l"(cx.t + imin(kn + lane, L - 1)));
                        asm volatile("prefetch.global.L1 [%0];" ::"l"(cx.t + imin(kn + 32 + lane, L - 1)));
                    }
                    if (cx.pe) {
#pragma unroll
                        for (int hc2 = 0; hc2 < 2; ++hc2) {
                            const int d0 = qp - (kn + 32 * hc2);
                            const int bd = d0 < -64 ? -64 : (d0 > L + 64 ? L + 64 : d0);
                            const int i0 = bd - 1 + kPosOff;
                            const float* p = cx.pe - kPosOff + (i0 & 1) * cx.Lt + (i0 & ~1);
                            asm volatile("prefetch.global.L1 [%0];" ::"l"(p - 30));
                            asm volatile("prefetch.global.L1 [%0];" ::"l"(p + 1));
                        }
                    }
                }"""
PATCHES = [("attn_fwd_sm100.cu", OLD, NEW)]
