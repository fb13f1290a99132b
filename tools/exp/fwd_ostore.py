# fwd: O rows leave through TMA stores of per-warp 32 x 32 bf16 boxes (64B-swizzled staging in the
# 32 KB freed by going from six to five K/V stages) instead of four 16-byte stores per thread and
# row; boxes that cross the sequence end (rows >= L) keep the per-row stores
OLD_ST = "constexpr int STAGES = 6;"
NEW_ST = "constexpr int STAGES = 5;"
OLD_SM = "constexpr int SMEM_BYTES = QT + STAGES * 2 * KT + 256 + 1024 + 512;"
NEW_SM = "constexpr int SMEM_BYTES = QT + STAGES * 2 * KT + 16 * 2048 + 256 + 1024 + 512;"
OLD_SIG = """attn_fwd_sm100(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
               const __grid_constant__ CUtensorMap tmV, AttnArgs a) {"""
NEW_SIG = """attn_fwd_sm100(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
               const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmO, AttnArgs a) {"""
OLD_TS = "    float* ts_s = reinterpret_cast<float*>(sKV + STAGES * 2 * KT);   // time_bias / 2 [32]"
NEW_TS = """    uint8_t* sO = sKV + STAGES * 2 * KT;           // 16 x 2 KB O staging boxes (one per epilogue warp)
    float* ts_s = reinterpret_cast<float*>(sO + 16 * 2048);   // time_bias / 2 [32]"""
OLD_O = """            UH_CHECK(!qok || (int64_t)o + qp < a.T);
            if (qok) {"""
NEW_O = """            UH_CHECK(!qok || (int64_t)o + qp < a.T);
            if (q0 + 32 * wq + 31 < L) {   // warp-uniform: the whole 32-row box lies inside the sequence
                uint8_t* box = sO + (warp - 4) * 2048;
                if (lane == 0) bulk_wait_read0();   // the previous item's store has read the box
                __syncwarp();
                const float sN = a.inv_n;
#pragma unroll
                for (int c = 0; c < 4; ++c)
                    *reinterpret_cast<uint4*>(box + lane * 64 + ((c ^ ((lane >> 1) & 3)) << 4)) =
                        make_uint4(pack_bf16(ov[c * 8 + 0] * sN, ov[c * 8 + 1] * sN),
                                   pack_bf16(ov[c * 8 + 2] * sN, ov[c * 8 + 3] * sN),
                                   pack_bf16(ov[c * 8 + 4] * sN, ov[c * 8 + 5] * sN),
                                   pack_bf16(ov[c * 8 + 6] * sN, ov[c * 8 + 7] * sN));
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) {
                    tma_store_2d(&tmO, box, h * DH + wg * 32, o + q0 + 32 * wq);
                    bulk_commit();
                }
            } else if (qok) {"""
OLD_END = """    __syncthreads();
    if (warp == 2) tmem_dealloc<512>(tmem);
}"""
NEW_END = """    if (warp >= 4 && lane == 0) bulk_wait0();   // O stores complete before the CTA retires
    __syncthreads();
    if (warp == 2) tmem_dealloc<512>(tmem);
}"""
OLD_L = """    UH_TRY(make_tmap_bf16(&tv, a.v, width, (uint64_t)T, a.ld_qkv, 64, BN));"""
NEW_L = """    UH_TRY(make_tmap_bf16(&tv, a.v, width, (uint64_t)T, a.ld_qkv, 64, BN));
    CUtensorMap to;   // O boxes: 32 columns x 32 rows, 64-byte swizzle
    UH_TRY(make_tmap_bf16(&to, a.out, width, (uint64_t)T, a.ld_out, 32, 32, 64));"""
PATCHES = [("attn_fwd_sm100.cu", OLD_ST, NEW_ST), ("attn_fwd_sm100.cu", OLD_SM, NEW_SM),
           ("attn_fwd_sm100.cu", OLD_SIG, NEW_SIG), ("attn_fwd_sm100.cu", OLD_TS, NEW_TS),
           ("attn_fwd_sm100.cu", OLD_O, NEW_O), ("attn_fwd_sm100.cu", OLD_END, NEW_END),
           ("attn_fwd_sm100.cu", OLD_L, NEW_L),
           ("attn_fwd_sm100.cu", "attn_fwd_sm100<<<grid, NUM_THREADS, SMEM_BYTES, st>>>(tq, tk, tv, a);",
            "attn_fwd_sm100<<<grid, NUM_THREADS, SMEM_BYTES, st>>>(tq, tk, tv, to, a);")]
