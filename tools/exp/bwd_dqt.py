# bwd: the fp32 dQ accumulator transposed ([H dh][T_pad], T_pad = T rounded up to 4): each dQ
# warp stages its [32 dh][32 q] box as 8 16-byte stores per thread (128B-swizzled) instead of 32
# scalar stores; dq_finish_k transposes through shared memory on the way to dQ
STAGE_OLD = """                for (int q = 0; q < 32; ++q) stg[q * 32 + lane] = v[q];
                fence_proxy_async_smem();
                __syncwarp();
                UH_CHECK(qb0 + 32 * hf < L + BN && h < a.H);
                if (lane == 0) {
                    tma_reduce_add_2d(&tmDQ, stg, h * DH + 32 * wq, o + qb0 + 32 * hf);"""
STAGE_NEW = """                for (int c = 0; c < 8; ++c)   // row lane (= dh), 16-byte chunk c, 128B swizzle
                    *reinterpret_cast<float4*>(reinterpret_cast<uint8_t*>(stg) + lane * 128 + ((c ^ (lane & 7)) << 4)) =
                        make_float4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
                fence_proxy_async_smem();
                __syncwarp();
                UH_CHECK(qb0 + 32 * hf < L + BN && h < a.H);
                if (lane == 0) {
                    tma_reduce_add_2d(&tmDQ, stg, o + qb0 + 32 * hf, h * DH + 32 * wq);"""
FIN_OLD = """// dQ = alpha/(2N) * acc (x gate), bf16, into its slice of dH
__global__ void __launch_bounds__(256) dq_finish_k(int64_t T, int width, const float* __restrict__ acc, int64_t lda,
                                                   const __nv_bfloat16* __restrict__ gate, int64_t ldg, float scale,
                                                   __nv_bfloat16* __restrict__ dq, int64_t ldq) {"""
FIN_NEW = """// dQ = alpha/(2N) * acc^T (x gate), bf16, into its slice of dH: 32-query x 64-dh tiles through
// shared memory (reads coalesced along T, writes along dh)
__global__ void __launch_bounds__(256) dq_finish_t_k(int64_t T, int width, const float* __restrict__ acc, int64_t lda,
                                                     const __nv_bfloat16* __restrict__ gate, int64_t ldg, float scale,
                                                     __nv_bfloat16* __restrict__ dq, int64_t ldq) {
    __shared__ float tile[64][33];
    const int tid = threadIdx.x;
    const int64_t nt = (T + 31) / 32;
    const int nd = width / 64;
    for (int64_t b = blockIdx.x; b < nt * nd; b += gridDim.x) {
        const int64_t t0 = (b / nd) * 32;
        const int d0 = (int)(b % nd) * 64;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int dr = k * 8 + (tid >> 5), tc = tid & 31;
            tile[dr][tc] = t0 + tc < T ? __ldcs(acc + (int64_t)(d0 + dr) * lda + t0 + tc) : 0.f;
        }
        __syncthreads();
        const int tr = tid >> 3, dc = (tid & 7) * 8;
        const int64_t row = t0 + tr;
        if (row < T) {
            float v[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) v[e] = tile[dc + e][tr] * scale;
            if (gate) {
                const uint4 gv = __ldg(reinterpret_cast<const uint4*>(gate + row * ldg + d0 + dc));
                const __nv_bfloat162* g2 = reinterpret_cast<const __nv_bfloat162*>(&gv);
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const float2 f = __bfloat1622float2(g2[e]);
                    v[2 * e] *= f.x; v[2 * e + 1] *= f.y;
                }
            }
            *reinterpret_cast<uint4*>(dq + row * ldq + d0 + dc) =
                make_uint4(pack_bf16(v[0], v[1]), pack_bf16(v[2], v[3]), pack_bf16(v[4], v[5]), pack_bf16(v[6], v[7]));
        }
        __syncthreads();
    }
}

// dQ = alpha/(2N) * acc (x gate), bf16, into its slice of dH
__global__ void __launch_bounds__(256) dq_finish_k(int64_t T, int width, const float* __restrict__ acc, int64_t lda,
                                                   const __nv_bfloat16* __restrict__ gate, int64_t ldg, float scale,
                                                   __nv_bfloat16* __restrict__ dq, int64_t ldq) {"""
LAUNCH_OLD = """    UH_TRY(make_tmap_f32(&dqm, akv.dq_acc, width, T, akv.ld_acc, 32, 32));
    UH_CUDA(cudaMemsetAsync(akv.dq_acc, 0, (size_t)T * akv.ld_acc * sizeof(float), st));"""
LAUNCH_NEW = """    const int64_t ldT = (T + 3) & ~int64_t(3);   // acc^T [width][ldT]
    UH_TRY(make_tmap_f32(&dqm, akv.dq_acc, (uint64_t)T, width, ldT, 32, 32, 128));
    UH_CUDA(cudaMemsetAsync(akv.dq_acc, 0, (size_t)width * ldT * sizeof(float), st));"""
FL_OLD = """    fb::dq_finish_k<<<4 * sms, 256, 0, st>>>(T, (int)width, akv.dq_acc, akv.ld_acc,"""
FL_NEW = """    fb::dq_finish_t_k<<<4 * sms, 256, 0, st>>>(T, (int)width, akv.dq_acc, ldT,"""
WS_OLD = """        off += align256((size_t)jag->total_tokens * desc->num_heads * desc->head_dim * sizeof(float));"""
WS_NEW = """        off += align256((size_t)((jag->total_tokens + 3) & ~int64_t(3)) * desc->num_heads * desc->head_dim * sizeof(float));"""
TM_OLD = """uh_status make_tmap_f32(CUtensorMap* map, const void* ptr, uint64_t inner, uint64_t outer, uint64_t ld_elems,
                        uint32_t box_inner, uint32_t box_outer) {"""
TM_NEW = """uh_status make_tmap_f32(CUtensorMap* map, const void* ptr, uint64_t inner, uint64_t outer, uint64_t ld_elems,
                        uint32_t box_inner, uint32_t box_outer, int swizzle_bytes) {"""
TM2_OLD = """    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,"""
TM2_NEW = """    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE,
                     swizzle_bytes == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B,"""
H_OLD = """uh_status make_tmap_f32(CUtensorMap* map, const void* ptr, uint64_t inner, uint64_t outer, uint64_t ld_elems,
                        uint32_t box_inner, uint32_t box_outer);"""
H_NEW = """uh_status make_tmap_f32(CUtensorMap* map, const void* ptr, uint64_t inner, uint64_t outer, uint64_t ld_elems,
                        uint32_t box_inner, uint32_t box_outer, int swizzle_bytes = 0);"""
PATCHES = [("attn_bwd_sm100.cu", STAGE_OLD, STAGE_NEW), ("attn_bwd_sm100.cu", FIN_OLD, FIN_NEW),
           ("attn_bwd_sm100.cu", LAUNCH_OLD, LAUNCH_NEW), ("attn_bwd_sm100.cu", FL_OLD, FL_NEW),
           ("attn.cu", WS_OLD, WS_NEW), ("runtime.cu", TM_OLD, TM_NEW), ("runtime.cu", TM2_OLD, TM2_NEW),
           ("internal.h", H_OLD, H_NEW)]
