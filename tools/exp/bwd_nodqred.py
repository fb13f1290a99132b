# backward: the dQ warps read dQ^T from TMEM but skip the shared staging + TMA reduction
PATCHES = [("attn_bwd_sm100.cu",
            "                if (lane == 0) bulk_wait_read0();\n                __syncwarp();\n#pragma unroll\n                for (int q = 0; q < BN; ++q) stg[q * 32 + lane] = v[q];",
            "                if (v[0] == 12345.678f) stg[lane] = v[1];\n                if (false) {\n#pragma unroll\n                for (int q = 0; q < BN; ++q) stg[q * 32 + lane] = v[q];"),
           ("attn_bwd_sm100.cu",
            "                    tma_reduce_add_2d(&tmDQ, stg, h * DH + 32 * wq, o + qb0);\n                    bulk_commit();\n                }",
            "                    tma_reduce_add_2d(&tmDQ, stg, h * DH + 32 * wq, o + qb0);\n                    bulk_commit();\n                }\n                }")]
