# bwd E1 + E2: one poller per role, the other warps of the role sleep in a named barrier
import runpy, os
base = runpy.run_path(os.path.join(os.path.dirname(os.path.abspath(__file__)), "bwd_e2bar.py"))
OLD = """                mbar_wait_sleep(&bars->s_full[sb], (sc >> 1) & 1);
                __syncwarp();   // tcgen05.ld is .sync.aligned: reconverge after the per-lane wait loop"""
NEW = """                if (warp == 4) mbar_wait_sleep(&bars->s_full[sb], (sc >> 1) & 1);
                __syncwarp();   // tcgen05.ld is .sync.aligned: reconverge after the per-lane wait loop
                named_bar_sync(6, 256);"""
PATCHES = base["PATCHES"] + [("attn_bwd_sm100.cu", OLD, NEW)]
