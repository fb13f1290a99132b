# bwd E1: timestamps a step ahead + the step's bias (classification, position pairs) formed before
# the S wait; after the TMEM load only h = alpha/2 S + bias remains (no cross-step registers)
import runpy, os
base = runpy.run_path(os.path.join(os.path.dirname(os.path.abspath(__file__)), "bwd_e1pipe.py"))
OLD = """            for (int i = 0; i < n; ++i, ++sc) {
                const int sb = sc & 1;
                const int qb = (k0 / BN + i) * BN + 32 * wg;   // this warpgroup's 32 queries
                const int32_t tcur = col_time(cx, qb, lane);
                const Chunk ch = k_chunk(cx, kp, kok, tk, qb, tcur);
                mbar_wait_sleep(&bars->s_full[sb], (sc >> 1) & 1);"""
NEW = """            int32_t t_nxt = col_time(cx, (k0 / BN) * BN + 32 * wg, lane);
            for (int i = 0; i < n; ++i, ++sc) {
                const int sb = sc & 1;
                const int qb = (k0 / BN + i) * BN + 32 * wg;   // this warpgroup's 32 queries
                const int32_t tcur = t_nxt;
                if (i + 1 < n) t_nxt = col_time(cx, qb + BN, lane);   // next step's, a step ahead
                const Chunk ch = k_chunk(cx, kp, kok, tk, qb, tcur);
                float hx[32];
                {
                    float2 pe2[16];
                    k_pos_issue(cx, ch, pe2);
                    k_bias(cx, ch, tk, pe2, hx);
                }
                mbar_wait_sleep(&bars->s_full[sb], (sc >> 1) & 1);"""
PATCHES = [base["PATCHES"][0], ("attn_bwd_sm100.cu", OLD, NEW), base["PATCHES"][2]]
