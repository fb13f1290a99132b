# backward: skip the FLAG_T1 masked sum of the d time_bias runs
PATCHES = [("attn_bwd_sm100.cu", "                        if (ch.flags & FLAG_T1) {   // columns [n, 32) are in bucket b_other\n                            float m[32];",
            "                        if (false) {   // columns [n, 32) are in bucket b_other\n                            float m[32];")]
