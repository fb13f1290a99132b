# GEMM residual epilogue: the 64-byte residual row segment per thread as two 32-byte loads
# (ld.global.nc.v8) instead of four 16-byte ones when the residual's stride allows
OLD = """                if (use_res) {
                    const uint4* rp = reinterpret_cast<const uint4*>(g.resid + (int64_t)row * g.ldr + col);
#pragma unroll
                    for (int j = 0; j < 4; ++j) rv4[j] = __ldg(rp + j);
                }"""
NEW = """                if (use_res) {
                    const __nv_bfloat16* rp = g.resid + (int64_t)row * g.ldr + col;
                    if (((reinterpret_cast<uintptr_t>(g.resid) | (uintptr_t)(g.ldr * 2)) & 31) == 0) {
#pragma unroll
                        for (int j = 0; j < 4; j += 2)
                            asm volatile("ld.global.nc.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                                         : "=r"(rv4[j].x), "=r"(rv4[j].y), "=r"(rv4[j].z), "=r"(rv4[j].w),
                                           "=r"(rv4[j + 1].x), "=r"(rv4[j + 1].y), "=r"(rv4[j + 1].z),
                                           "=r"(rv4[j + 1].w)
                                         : "l"(rp + j * 8));
                    } else {
#pragma unroll
                        for (int j = 0; j < 4; ++j) rv4[j] = __ldg(reinterpret_cast<const uint4*>(rp) + j);
                    }
                }"""
PATCHES = [("gemm_sm100.cuh", OLD, NEW)]
