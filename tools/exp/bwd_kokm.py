# bwd: keys beyond L handled by the chunk's FLAG_M visibility mask instead of per-element selects
PATCHES = [
    ("attn_common.cuh", "r.flags = __reduce_or_sync(0xffffffffu, kok ? f : 0u);",
     "r.flags = __reduce_or_sync(0xffffffffu, kok ? f : (unsigned)FLAG_M);"),
    ("attn_bwd_sm100.cu", """                    d2[c] = kok ? pack_bf16(dv.x, dv.y) : 0u;   // keys beyond L must not reach dQ
                    dp[2 * c] = kok ? dv.x : 0.f;                // dp now holds the fp32 dS'
                    dp[2 * c + 1] = kok ? dv.y : 0.f;""",
     """                    d2[c] = pack_bf16(dv.x, dv.y);
                    dp[2 * c] = dv.x;
                    dp[2 * c + 1] = dv.y;"""),
]
