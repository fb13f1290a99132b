# bwd dQ warps: p_full probed right after dq_full, and ds_free released as soon as the dS^T row is
# in registers (before the diagonal sums), so the P/dS warps' store two steps later never waits
import os, runpy
base = runpy.run_path(os.path.join(os.path.dirname(os.path.abspath(__file__)), "bwd_e2ptest.py"))["PATCHES"]
OLD = """                        uint32_t d2[16];
#pragma unroll
                        for (int c = 0; c < 4; ++c) {
                            const uint4 u = *reinterpret_cast<const uint4*>(row + (((4 * hf + c) ^ (r & 7)) << 4));
                            d2[4 * c] = u.x; d2[4 * c + 1] = u.y; d2[4 * c + 2] = u.z; d2[4 * c + 3] = u.w;
                        }
                        if (C - 31 >= a.P - 1) {"""
NEW = """                        uint32_t d2[16];
#pragma unroll
                        for (int c = 0; c < 4; ++c) {
                            const uint4 u = *reinterpret_cast<const uint4*>(row + (((4 * hf + c) ^ (r & 7)) << 4));
                            d2[4 * c] = u.x; d2[4 * c + 1] = u.y; d2[4 * c + 2] = u.z; d2[4 * c + 3] = u.w;
                        }
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&bars->ds_free[sb]);   // the row is in registers
                        ds_done = true;
                        if (C - 31 >= a.P - 1) {"""
OLD2 = """                __syncwarp();
                if (lane == 0) mbar_arrive(&bars->ds_free[sb]);
                if (warp == 12) TRACE_FB(6, sc);"""
NEW2 = """                __syncwarp();
                if (!ds_done && lane == 0) mbar_arrive(&bars->ds_free[sb]);
                if (warp == 12) TRACE_FB(6, sc);"""
OLD3 = """                if (a.dpos) {
                    // d pos_bias[min(q - k, P - 1)] += ds"""
NEW3 = """                bool ds_done = false;   // warp-uniform
                if (a.dpos) {
                    // d pos_bias[min(q - k, P - 1)] += ds"""
PATCHES = base + [("attn_bwd_sm100.cu", OLD, NEW), ("attn_bwd_sm100.cu", OLD2, NEW2), ("attn_bwd_sm100.cu", OLD3, NEW3)]
