# trace build: item-boundary timeline of the forward (event 6: warp 4 past the o_full wait,
# event 7: warp 4 after the O read-out and o_empty; the MMA warp's ring take is event 5's slot)
FLAGS = ["-DUH_TRACE=1"]
PATCHES = [
    ("attn_fwd_sm100.cu", "                    TRACE(7 * 1024 + (kc & 1023));   // stage free: PV(kc - STAGES) done\n", ""),
    ("attn_fwd_sm100.cu", "                if (warp == 8 && lane == 0) TRACE(6 * 1024 + (sc & 1023));\n", ""),
    ("attn_fwd_sm100.cu", """            mbar_wait_sleep(&bars->o_full, qi & 1);
            tc_fence_after();""", """            mbar_wait_sleep(&bars->o_full, qi & 1);
            if (warp == 4 && lane == 0) TRACE(6 * 1024 + (sc & 1023));
            tc_fence_after();"""),
    ("attn_fwd_sm100.cu", """            if (lane == 0) mbar_arrive(&bars->o_empty);""", """            if (lane == 0) mbar_arrive(&bars->o_empty);
            if (warp == 4 && lane == 0) TRACE(7 * 1024 + (sc & 1023));"""),
]
