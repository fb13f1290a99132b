# trace build: event 6 = warp 4 after the O read-out (o_empty), event 7 = warp 4 after the next
# item's setup (ChunkCtx, row timestamp), before its first tile
FLAGS = ["-DUH_TRACE=1"]
PATCHES = [
    ("attn_fwd_sm100.cu", "                    TRACE(7 * 1024 + (kc & 1023));   // stage free: PV(kc - STAGES) done\n", ""),
    ("attn_fwd_sm100.cu", "                if (warp == 8 && lane == 0) TRACE(6 * 1024 + (sc & 1023));\n", ""),
    ("attn_fwd_sm100.cu", """            if (lane == 0) mbar_arrive(&bars->o_empty);""", """            if (lane == 0) mbar_arrive(&bars->o_empty);
            if (warp == 4 && lane == 0) TRACE(6 * 1024 + (sc & 1023));"""),
    ("attn_fwd_sm100.cu", """            const int32_t tq = (a.ts && qok) ? rel32(tqn, cx.t0) : 0;""",
     """            const int32_t tq = (a.ts && qok) ? rel32(tqn, cx.t0) : 0;
            if (warp == 4 && lane == 0) TRACE(7 * 1024 + ((sc + (tq & 0) + (int)(cx.pos_far * 0.f)) & 1023));"""),
]
