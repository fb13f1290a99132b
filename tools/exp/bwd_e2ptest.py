# bwd dQ warps: probe p_full (test_wait, acquire) right after dq_full instead of a blocking wait
# just before the dS^T reads, so its latency overlaps the dQ^T read-out and staging
PATCHES = [
    ("attn_bwd_sm100.cu", """                mbar_wait_sleep(&bars->dq_full[sb], (sc >> 1) & 1);
                __syncwarp();
                if (warp == 12) TRACE_FB(5, sc);""", """                mbar_wait_sleep(&bars->dq_full[sb], (sc >> 1) & 1);
                const bool pf_rdy = mbar_test(smem_u32(&bars->p_full[sb]), (sc >> 1) & 1);
                __syncwarp();
                if (warp == 12) TRACE_FB(5, sc);"""),
    ("attn_bwd_sm100.cu", "mbar_wait(&bars->p_full[sb], (sc >> 1) & 1);   // the P/dS warps' shared stores are visible",
     "if (!pf_rdy) mbar_wait(&bars->p_full[sb], (sc >> 1) & 1);   // the P/dS warps' shared stores are visible"),
]
