# bisect: no d pos_bias work in the dQ warps
PATCHES = [("attn_bwd_sm100.cu", "                if (a.dpos) {\n                    // d pos_bias[min(q - k, P - 1)] += ds",
            "                if (false) {\n                    // d pos_bias[min(q - k, P - 1)] += ds")]
