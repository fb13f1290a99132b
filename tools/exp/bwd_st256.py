# bwd dV / dK rows: 32-byte gate loads and stores (ld/st.global.v8.b32) when the row stride allows
OLD = """    if (gate) {
        const uint4* g = reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(gate) + row * ldg + col);
#pragma unroll
        for (int ch = 0; ch < 8; ++ch) {
            uint4 gv = __ldg(g + ch);
            const __nv_bfloat162* g2 = reinterpret_cast<const __nv_bfloat162*>(&gv);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                float2 f = __bfloat1622float2(g2[e]);
                w[ch * 8 + 2 * e] *= f.x;
                w[ch * 8 + 2 * e + 1] *= f.y;
            }
        }
    }
    uint4* o = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(base) + row * ld + col);
#pragma unroll
    for (int ch = 0; ch < 8; ++ch)
        o[ch] = make_uint4(pack_bf16(w[ch * 8 + 0], w[ch * 8 + 1]), pack_bf16(w[ch * 8 + 2], w[ch * 8 + 3]),
                           pack_bf16(w[ch * 8 + 4], w[ch * 8 + 5]), pack_bf16(w[ch * 8 + 6], w[ch * 8 + 7]));
}"""
NEW = """    const bool v8 = ((reinterpret_cast<uintptr_t>(base) | (uintptr_t)(ld * 2) |
                      (gate ? (reinterpret_cast<uintptr_t>(gate) | (uintptr_t)(ldg * 2)) : 0)) & 31) == 0;
    if (gate) {
        const __nv_bfloat16* gp = reinterpret_cast<const __nv_bfloat16*>(gate) + row * ldg + col;
#pragma unroll
        for (int ch = 0; ch < 8; ch += 2) {
            uint32_t gw[8];
            if (v8) {
                asm volatile("ld.global.nc.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                             : "=r"(gw[0]), "=r"(gw[1]), "=r"(gw[2]), "=r"(gw[3]), "=r"(gw[4]), "=r"(gw[5]),
                               "=r"(gw[6]), "=r"(gw[7]) : "l"(gp + ch * 8));
            } else {
                const uint4 a0 = __ldg(reinterpret_cast<const uint4*>(gp + ch * 8));
                const uint4 a1 = __ldg(reinterpret_cast<const uint4*>(gp + ch * 8 + 8));
                gw[0] = a0.x; gw[1] = a0.y; gw[2] = a0.z; gw[3] = a0.w;
                gw[4] = a1.x; gw[5] = a1.y; gw[6] = a1.z; gw[7] = a1.w;
            }
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const float2 f = unpack_bf16x2(gw[e]);
                w[ch * 8 + 2 * e] *= f.x;
                w[ch * 8 + 2 * e + 1] *= f.y;
            }
        }
    }
    __nv_bfloat16* op = reinterpret_cast<__nv_bfloat16*>(base) + row * ld + col;
#pragma unroll
    for (int ch = 0; ch < 8; ch += 2) {
        uint32_t p[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) p[e] = pack_bf16(w[ch * 8 + 2 * e], w[ch * 8 + 2 * e + 1]);
        if (v8) {
            asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(op + ch * 8), "r"(p[0]), "r"(p[1]),
                         "r"(p[2]), "r"(p[3]), "r"(p[4]), "r"(p[5]), "r"(p[6]), "r"(p[7]) : "memory");
        } else {
            *reinterpret_cast<uint4*>(op + ch * 8) = make_uint4(p[0], p[1], p[2], p[3]);
            *reinterpret_cast<uint4*>(op + ch * 8 + 8) = make_uint4(p[4], p[5], p[6], p[7]);
        }
    }
}"""
PATCHES = [("attn_bwd_sm100.cu", OLD, NEW)]
