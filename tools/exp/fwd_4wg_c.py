# fwd: four epilogue warpgroups (640 threads; setmaxnreg: control warpgroup 32, epilogue 112
# registers), four S buffers (S three tiles ahead of PV), tile j -> warpgroup j % 4 = buffer j % 4;
# the O epilogue split over the four warpgroups (32 columns each)
REG_CTRL, REG_EPI = 64, 104
O_OLD = """            // ---- O epilogue: A = O / N (warpgroups 0 and 1, 64 columns each)
            if (wg == 2) continue;
            mbar_wait_sleep(&bars->o_full, qi & 1);
            tc_fence_after();
            float ov[64];
            tmem_ld32(tmem + lane_base + O_COL + wg * 64, ov);
            tmem_ld32(tmem + lane_base + O_COL + wg * 64 + 32, ov + 32);
            tmem_ld_wait();"""
O_NEW = """            // ---- O epilogue: A = O / N (32 columns per warpgroup)
            mbar_wait_sleep(&bars->o_full, qi & 1);
            tc_fence_after();
            float ov[32];
            tmem_ld32(tmem + lane_base + O_COL + wg * 32, ov);
            tmem_ld_wait();"""
S_OLD = """                                                     (int64_t)(o + qp) * a.ld_out + h * DH + wg * 64);
                const float sN = a.inv_n;
#pragma unroll
                for (int ch = 0; ch < 8; ++ch)"""
S_NEW = """                                                     (int64_t)(o + qp) * a.ld_out + h * DH + wg * 32);
                const float sN = a.inv_n;
#pragma unroll
                for (int ch = 0; ch < 4; ++ch)"""
PATCHES = [
    ("attn_fwd_sm100.cu", "constexpr int NUM_THREADS = 512;", "constexpr int NUM_THREADS = 640;"),
    ("attn_fwd_sm100.cu", "constexpr int NS = 3;", "constexpr int NS = 4;"),
    ("attn_fwd_sm100.cu", "ring_init(&bars->ring, 13);   // MMA warp + 12 epilogue warps",
     "ring_init(&bars->ring, 17);"),
    ("attn_fwd_sm100.cu", "mbar_init(&bars->o_empty, 8);", "mbar_init(&bars->o_empty, 16);"),
    ("attn_fwd_sm100.cu", "if (sc % 3 != wg) continue;", "if ((sc & 3) != wg) continue;"),
    ("attn_fwd_sm100.cu", O_OLD, O_NEW),
    ("attn_fwd_sm100.cu", S_OLD, S_NEW),
    ("attn_fwd_sm100.cu", "    if (warp == 0) {\n",
     "    if (warp < 4) {\n    asm volatile(\"setmaxnreg.dec.sync.aligned.u32 %%0;\\n\" ::\"n\"(%d));\n    if (warp == 0) {\n" % REG_CTRL),
    ("attn_fwd_sm100.cu", "    } else if (warp >= 4) {\n",
     "    }\n    } else {\n        asm volatile(\"setmaxnreg.inc.sync.aligned.u32 %%0;\\n\" ::\"n\"(%d));\n" % REG_EPI),
]
