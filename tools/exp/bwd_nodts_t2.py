# backward: skip only the per-element (FLAG_T2) part of the d time_bias runs
PATCHES = [("attn_bwd_sm100.cu",
            "                        for (int j = 0; j < 32; ++j)\n                            run_add(bucket32(__shfl_sync(0xffffffffu, ch.tcol, j) - tk, cx.NB), dp[j]);",
            "                        for (int j = 0; j < 1; ++j)\n                            run_add(bucket32(__shfl_sync(0xffffffffu, ch.tcol, j) - tk, cx.NB), dp[j]);")]
