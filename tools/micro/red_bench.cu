// fp32 reduction throughput into a [262144 x 512] buffer (the fused attention backward's dQ
// accumulator) with the access pattern of key-major items: per item (sequence, head, 128-key
// tile) 20 steps of a [64 queries x 128 dh] fp32 block, starting at the key tile and moving
// forward.  Each of 8 warps reduces a [32 q x 32 dh] box per step.  Methods:
//   0: red.global.add.f32, lane = dh, 32 instructions (128 B per warp instruction)
//   1: red.global.add.v4.f32, 8 instructions (512 B per warp instruction)
//   2: st.shared box + cp.reduce.async.bulk.tensor.2d add (TMA), double-buffered per warp
#include <cstdint>
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>
#include "../../paper_2602_16986_b200/csrc/sm100.cuh"
using namespace uh;

constexpr int T = 262144, D = 512, STEPS = 20;

__device__ __forceinline__ uint32_t hash(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x;
}

template <int METHOD>
__global__ void __launch_bounds__(256, 1) k(float* acc, const __grid_constant__ CUtensorMap tm, int items, long long* cyc, int ordered) {
    extern __shared__ __align__(1024) float stg_raw[];
    float (*stg)[2][32 * 32] = reinterpret_cast<float (*)[2][32 * 32]>(stg_raw);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, wg = warp >> 2, wq = warp & 3;
    long long t0 = clock64();
    int buf = 0;
    for (int i = 0; i < items; ++i) {
        const uint32_t r = hash(blockIdx.x * 7919u + i * 104729u);
        int seq = r % 16, head = (r >> 4) % 4, tile = (r >> 8) % 128;
        if (ordered) {   // items in (sequence, key tile, head) order, taken round-robin by the CTAs
            const int g = i * gridDim.x + blockIdx.x;
            head = g % 4; tile = (g / 4) % 128; seq = (g / 512) % 16;
        }
        for (int s = 0; s < STEPS; ++s) {
            int q0 = tile * 128 + s * 64 + wg * 32;
            if (q0 + 32 > 16384) q0 = 16384 - 32;
            const int row0 = seq * 16384 + q0, col0 = head * 128 + wq * 32;
            const float v = (float)(lane + s);
            if (METHOD == 0) {
#pragma unroll
                for (int q = 0; q < 32; ++q)
                    asm volatile("red.global.add.f32 [%0], %1;" ::"l"(acc + (size_t)(row0 + q) * D + col0 + lane), "f"(v) : "memory");
            } else if (METHOD == 1) {
#pragma unroll
                for (int j = 0; j < 8; ++j) {   // 32 rows x 8 float4 = 256 vectors, 8 per lane
                    const int e = j * 32 + lane, q = e >> 3, c = (e & 7) * 4;
                    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(acc + (size_t)(row0 + q) * D + col0 + c),
                                 "f"(v), "f"(v), "f"(v), "f"(v) : "memory");
                }
            } else {
                float* box = stg[warp][buf];
                if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                __syncwarp();
#pragma unroll
                for (int q = 0; q < 32; ++q) box[q * 32 + lane] = v;
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if (lane == 0) {
                    asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile.bulk_group [%0, {%1, %2}], [%3];"
                                 ::"l"(&tm), "r"(col0), "r"(row0), "r"(smem_u32(box)) : "memory");
                    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                }
                buf ^= 1;
            }
        }
    }
    if (METHOD == 2 && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    __syncthreads();
    if (blockIdx.x == 0 && threadIdx.x == 0) cyc[0] = clock64() - t0;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <int M>
void run(float* acc, const CUtensorMap& tm, long long* o, int items, const char* name, int ordered) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaFuncSetAttribute(k<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    k<M><<<148, 256, 65536>>>(acc, tm, 4, o, ordered);
    cudaMemset(acc, 0, (size_t)T * D * 4);
    cudaEventRecord(e0);
    k<M><<<148, 256, 65536>>>(acc, tm, items, o, ordered);
    cudaEventRecord(e1);
    cudaDeviceSynchronize();
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double bytes = 148.0 * items * STEPS * 64 * 128 * 4;
    printf("%s %-24s %8.3f ms  %6.2f TB/s reduced (%.1f us per 32 KB step per SM)  %s\n", ordered ? "ordered" : "random ", name, ms, bytes / (ms * 1e-3) / 1e12,
           ms * 1e3 / (items * STEPS), cudaGetErrorString(cudaGetLastError()));
}

int main() {
    float* acc; cudaMalloc(&acc, (size_t)T * D * 4); cudaMemset(acc, 0, (size_t)T * D * 4);
    long long* o; cudaMalloc(&o, 64);
    EncodeFn enc; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
    CUtensorMap tm;
    cuuint64_t dims[2] = {D, T}, strides[1] = {D * 4};
    cuuint32_t box[2] = {32, 32}, es[2] = {1, 1};
    CUresult cr = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, acc, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode %d\n", (int)cr);
    for (int ord = 0; ord < 2; ++ord) {
        run<0>(acc, tm, o, 60, "red.f32 x32", ord);
        run<1>(acc, tm, o, 60, "red.v4.f32 x8", ord);
        run<2>(acc, tm, o, 60, "TMA reduce 32x32 box", ord);
    }
    return 0;
}
