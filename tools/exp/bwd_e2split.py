# bwd: the dQ warpgroups split by role (warpgroup 0: dQ^T read-out + staging + TMA reduce for both
# query halves; warpgroup 1: d pos_bias for both halves, from p_full instead of dq_full)
import os
H = os.path.dirname(os.path.abspath(__file__))
PATCHES = [("attn_bwd_sm100.cu", open(os.path.join(H, "bwd_e2split_old.cu.txt")).read(),
            open(os.path.join(H, "bwd_e2split.cu.txt")).read()),
           ("attn_bwd_sm100.cu", "mbar_init(&bars->s_free[i], 8); mbar_init(&bars->ds_free[i], 8);",
            "mbar_init(&bars->s_free[i], 4); mbar_init(&bars->ds_free[i], 4);")]
