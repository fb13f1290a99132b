# bwd P/dS warps: prefetch.global.L1 of the next query step's column timestamps and position-table
# pairs (the table does not stay in the ~30 KB of L1 left by the kernel's shared memory, so every
# step's pair loads otherwise come from L2); no registers are held across the step
OLD = """                const Chunk ch = k_chunk(cx, kp, kok, tk, qb, tcur);
                mbar_wait_sleep(&bars->s_full[sb], (sc >> 1) & 1);"""
NEW = """                const Chunk ch = k_chunk(cx, kp, kok, tk, qb, tcur);
                if (i + 1 < n) {   // next step: its timestamps and position pairs into L1
                    const int qn = qb + BN;
                    if (cx.ts_h) asm volatile("prefetch.global.L1 [%0];" ::"l"(cx.t + imin(qn + lane, L - 1)));
                    if (cx.pe) {
                        const int d0 = qn - kp;
                        const int bd = d0 < -96 ? -96 : (d0 > L + 64 ? L + 64 : d0);
                        const int i0 = bd + kPosOff;
                        const float* p = cx.pe - kPosOff + (i0 & 1) * cx.Lt + (i0 & ~1);
                        asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
                        asm volatile("prefetch.global.L1 [%0];" ::"l"(p + 31));
                    }
                }
                mbar_wait_sleep(&bars->s_full[sb], (sc >> 1) & 1);"""
PATCHES = [("attn_bwd_sm100.cu", OLD, NEW)]
