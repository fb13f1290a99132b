# bisect: second dQ warpgroup idle (first does queries 0-31 only)
PATCHES = [("attn_bwd_sm100.cu", "        const int wq = warp & 3, hf = (warp - 12) >> 2;",
            "        const int wq = warp & 3, hf = (warp - 12) >> 2;\n        if (hf == 1) { __syncwarp(); named_bar_sync(1, THREADS); return; }"),
           ("attn_bwd_sm100.cu", "mbar_init(&bars->s_free[i], 8); mbar_init(&bars->ds_free[i], 8);",
            "mbar_init(&bars->s_free[i], 4); mbar_init(&bars->ds_free[i], 4);"),
           ("attn_bwd_sm100.cu", "ring_init(&bars->ring, 18);", "ring_init(&bars->ring, 14);")]
