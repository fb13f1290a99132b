# fwd O epilogue: each thread's 64-byte row segment leaves as two 32-byte stores (STG.256) instead
# of four 16-byte ones (half the LSU requests of the uncoalesced row stores at item boundaries)
OLD = """            if (qok) {
                uint4* op = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(a.out) +
                                                     (int64_t)(o + qp) * a.ld_out + h * DH + wg * 32);
                const float sN = a.inv_n;
#pragma unroll
                for (int ch = 0; ch < 4; ++ch)"""
NEW = """            const bool v8 = ((reinterpret_cast<uintptr_t>(a.out) | (uintptr_t)(a.ld_out * 2)) & 31) == 0;
            if (qok && v8) {
                uint32_t* op = reinterpret_cast<uint32_t*>(reinterpret_cast<__nv_bfloat16*>(a.out) +
                                                           (int64_t)(o + qp) * a.ld_out + h * DH + wg * 32);
                const float sN = a.inv_n;
#pragma unroll
                for (int hv = 0; hv < 2; ++hv) {
                    uint32_t w8[8];
#pragma unroll
                    for (int e = 0; e < 8; ++e)
                        w8[e] = pack_bf16(ov[hv * 16 + 2 * e] * sN, ov[hv * 16 + 2 * e + 1] * sN);
                    asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(op + hv * 8),
                                 "r"(w8[0]), "r"(w8[1]), "r"(w8[2]), "r"(w8[3]), "r"(w8[4]), "r"(w8[5]), "r"(w8[6]),
                                 "r"(w8[7]) : "memory");
                }
            } else if (qok) {
                uint4* op = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(a.out) +
                                                     (int64_t)(o + qp) * a.ld_out + h * DH + wg * 32);
                const float sN = a.inv_n;
#pragma unroll
                for (int ch = 0; ch < 4; ++ch)"""
PATCHES = [("attn_fwd_sm100.cu", OLD, NEW)]
