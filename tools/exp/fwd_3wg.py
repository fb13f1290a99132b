# fwd: three epilogue warpgroups (512 threads, 128 registers each), tile j -> warpgroup j % 3 =
# S buffer j % 3, so three tiles' SiLU epilogues can be in flight (the MMA loop is unchanged)
PATCHES = [
    ("attn_fwd_sm100.cu", "constexpr int NUM_THREADS = 384;", "constexpr int NUM_THREADS = 512;"),
    ("attn_fwd_sm100.cu", "ring_init(&bars->ring, 9);   // MMA warp + 8 epilogue warps",
     "ring_init(&bars->ring, 13);   // MMA warp + 12 epilogue warps"),
    ("attn_fwd_sm100.cu", "if ((sc & 1) != wg) continue;", "if (sc % 3 != wg) continue;"),
    ("attn_fwd_sm100.cu", """            // ---- O epilogue: A = O / N
            mbar_wait_sleep(&bars->o_full, qi & 1);""", """            // ---- O epilogue: A = O / N (warpgroups 0 and 1, 64 columns each)
            if (wg == 2) continue;
            mbar_wait_sleep(&bars->o_full, qi & 1);"""),
]
