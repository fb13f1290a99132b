# fwd epilogue: wait for S with the plain try_wait loop instead of the suspend-hint variant
PATCHES = [("attn_fwd_sm100.cu", "mbar_wait_sleep(&bars->s_full[sb], (sc / NS) & 1);",
            "mbar_wait(&bars->s_full[sb], (sc / NS) & 1);")]
