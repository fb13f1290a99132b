# backward: skip the position-bias gradient (cost of the skewed diagonal sums)
PATCHES = [("attn_bwd_sm100.cu", "                if (a.dpos) {\n                    // d pos_bias[min(q - k, P - 1)] += ds", "                if (false) {\n                    // d pos_bias[min(q - k, P - 1)] += ds")]
