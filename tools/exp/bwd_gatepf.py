# bwd P/dS warps, item end: the dV gate row (silu'(h_V), 64 bf16) is loaded before the acc_full
# wait (the dK gate row after acc_empty), so no global load sits between the dV and dK TMEM
# reads that release the accumulators (acc_empty) for the next item
HELPERS = r'''
// 64 bf16 gate values of a row (32 packed words), 32-byte loads when aligned
__device__ __forceinline__ void load_gate64(const void* gate, int64_t ldg, int64_t row, int col, bool v8, uint32_t* g) {
    const __nv_bfloat16* gp = reinterpret_cast<const __nv_bfloat16*>(gate) + row * ldg + col;
#pragma unroll
    for (int ch = 0; ch < 8; ch += 2) {
        uint32_t* gw = g + ch * 4;
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
    }
}
// row of 32 values x scale (x gate when given) -> bf16, 32-byte stores when aligned
__device__ __forceinline__ void store_row32_g(void* base, int64_t ld, int64_t row, int col, const float* v,
                                              const uint32_t* g, float scale, bool v8) {
    __nv_bfloat16* op = reinterpret_cast<__nv_bfloat16*>(base) + row * ld + col;
#pragma unroll
    for (int ch = 0; ch < 4; ch += 2) {
        uint32_t p[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            float a0 = v[ch * 8 + 2 * e] * scale, a1 = v[ch * 8 + 2 * e + 1] * scale;
            if (g) { const float2 f = unpack_bf16x2(g[ch * 4 + e]); a0 *= f.x; a1 *= f.y; }
            p[e] = pack_bf16(a0, a1);
        }
        if (v8) {
            asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(op + ch * 8), "r"(p[0]), "r"(p[1]),
                         "r"(p[2]), "r"(p[3]), "r"(p[4]), "r"(p[5]), "r"(p[6]), "r"(p[7]) : "memory");
        } else {
            *reinterpret_cast<uint4*>(op + ch * 8) = make_uint4(p[0], p[1], p[2], p[3]);
            *reinterpret_cast<uint4*>(op + ch * 8 + 8) = make_uint4(p[4], p[5], p[6], p[7]);
        }
    }
}
'''
OLD = """            mbar_wait_sleep(&bars->acc_full, ki & 1);
            __syncwarp();
            tc_fence_after();
            {   // dV then dK (64 registers at a time under the 512-thread register budget)
                float acc[64];
                tmem_ld32(tmem + lane_base + DV_COL + wg * 64, acc);
                tmem_ld32(tmem + lane_base + DV_COL + wg * 64 + 32, acc + 32);
                tmem_ld_wait();
                UH_CHECK(!kok || o + kp < a.T);
                if (kok) store_out_row64(a.dv, a.ld_grad, o + kp, h * DH + wg * 64, acc, a.gv, a.ld_gate, a.inv_n);
                tmem_ld32(tmem + lane_base + DK_COL + wg * 64, acc);
                tmem_ld32(tmem + lane_base + DK_COL + wg * 64 + 32, acc + 32);
                tmem_ld_wait();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&bars->acc_empty);
                if (kok) store_out_row64(a.dk, a.ld_grad, o + kp, h * DH + wg * 64, acc, a.gk, a.ld_gate, ha * a.inv_n);
            }"""
NEW = """            const bool v8 = ((reinterpret_cast<uintptr_t>(a.dv) | reinterpret_cast<uintptr_t>(a.dk) |
                              (uintptr_t)(a.ld_grad * 2) | reinterpret_cast<uintptr_t>(a.gv) |
                              reinterpret_cast<uintptr_t>(a.gk) | (uintptr_t)(a.ld_gate * 2)) & 31) == 0;
            uint32_t gw[32];
            if (kok && a.gv) load_gate64(a.gv, a.ld_gate, o + kp, h * DH + wg * 64, v8, gw);   // hides behind the wait
            mbar_wait_sleep(&bars->acc_full, ki & 1);
            __syncwarp();
            tc_fence_after();
            UH_CHECK(!kok || o + kp < a.T);
#pragma unroll 1
            for (int hh = 0; hh < 2; ++hh) {   // dV, 32 columns at a time
                float acc[32];
                tmem_ld32(tmem + lane_base + DV_COL + wg * 64 + 32 * hh, acc);
                tmem_ld_wait();
                if (kok) store_row32_g(a.dv, a.ld_grad, o + kp, h * DH + wg * 64 + 32 * hh, acc,
                                       a.gv ? gw + 16 * hh : nullptr, a.inv_n, v8);
            }
            {
                float acc[64];
                tmem_ld32(tmem + lane_base + DK_COL + wg * 64, acc);
                tmem_ld32(tmem + lane_base + DK_COL + wg * 64 + 32, acc + 32);
                tmem_ld_wait();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&bars->acc_empty);
                if (kok && a.gk) load_gate64(a.gk, a.ld_gate, o + kp, h * DH + wg * 64, v8, gw);
                if (kok) {
                    store_row32_g(a.dk, a.ld_grad, o + kp, h * DH + wg * 64, acc, a.gk ? gw : nullptr, ha * a.inv_n, v8);
                    store_row32_g(a.dk, a.ld_grad, o + kp, h * DH + wg * 64 + 32, acc + 32, a.gk ? gw + 16 : nullptr,
                                  ha * a.inv_n, v8);
                }
            }"""
PATCHES = [("attn_bwd_sm100.cu", "// sum of 32 fp32 values as a tree of packed FADD2", HELPERS + "\n// sum of 32 fp32 values as a tree of packed FADD2"),
           ("attn_bwd_sm100.cu", OLD, NEW)]
