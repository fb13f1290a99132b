# measurement only (wrong d pos_bias): the dQ warps skip the d pos_bias diagonal sums
PATCHES = [("attn_bwd_sm100.cu", "                if (a.dpos) {\n                    // d pos_bias[min(q - k, P - 1)] += ds", "                if (false) {\n                    // d pos_bias[min(q - k, P - 1)] += ds")]
