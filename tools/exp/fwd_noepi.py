# forward: the epilogue releases P without computing it (MMA + load throughput alone)
PATCHES = [("attn_fwd_sm100.cu",
            "                tc_fence_after();\n#pragma unroll\n                for (int hc = 0; hc < 2; ++hc) {",
            "                tc_fence_after();\n                if (lane == 0) mbar_arrive(&bars->p_full[sb]);\n                continue;\n#pragma unroll\n                for (int hc = 0; hc < 2; ++hc) {")]
