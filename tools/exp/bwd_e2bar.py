# bwd E2: one dQ warp polls dq_full, the other seven sleep in a named barrier (no polling loops
# taking issue slots from the P/dS warps on the same sub-partitions)
OLD = """                mbar_wait_sleep(&bars->dq_full[sb], (sc >> 1) & 1);
                __syncwarp();
                if (warp == 12) TRACE_FB(5, sc);"""
NEW = """                if (warp == 12) mbar_wait_sleep(&bars->dq_full[sb], (sc >> 1) & 1);
                __syncwarp();
                named_bar_sync(5, 256);
                if (warp == 12) TRACE_FB(5, sc);"""
PATCHES = [("attn_bwd_sm100.cu", OLD, NEW)]
