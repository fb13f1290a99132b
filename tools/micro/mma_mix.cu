// The dK/dV kernel's per-step MMA mix without TMA or epilogue: 16 SS MMAs (M=128, N=64; A = K or V
// 32 KB tiles, B = Q or dA 16 KB tiles, both K-major SW128) into two TMEM accumulators, then 8 TS
// MMAs (M=128, N=128; A from TMEM, B MN-major) into two more.  Cycles per step vs the floor 1280.
// Variants isolate the SS part, the TS part, and the SS part with a single accumulator.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2602_16986_b200/csrc/sm100.cuh"
using namespace uh;

constexpr int KT = 32768, QT = 16384;

__global__ void __launch_bounds__(128, 1) k(long long* out, int steps, int mode) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    __shared__ uint32_t slot;
    __shared__ __align__(8) uint64_t done;
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < (2 * KT + 2 * QT) / 4; i += blockDim.x) ((uint32_t*)smem)[i] = 0x3c003c00u ^ (i * 2654435761u & 0x00ff00ffu);
    if (threadIdx.x == 0) { mbar_init(&done, 1); fence_barrier_init(); }
    if (warp == 2) tmem_alloc<512>(&slot);
    fence_proxy_async_smem();
    tc_fence_before(); __syncthreads(); tc_fence_after();
    const uint32_t tmem = slot;
    if (warp == 1) {
        constexpr uint32_t idesc_s = make_idesc_bf16(128, 64, false, false);
        constexpr uint32_t idesc_a = make_idesc_bf16(128, 128, false, true);
        const uint64_t dk = make_sw128_desc(smem_u32(smem), 16, 1024), dv = dk + (KT >> 4);
        const uint64_t dq = make_sw128_desc(smem_u32(smem) + 2 * KT, 16, 1024), dda = dq + (QT >> 4);
        const uint64_t qmn = make_sw128_desc(smem_u32(smem) + 2 * KT, QT / 2, 1024), damn = qmn + (QT >> 4);
        long long t0 = clock64();
        for (int s = 0; s < steps; ++s) {
            const int sb = s & 1;
            if (elect_one()) {
                if (mode != 2) {
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk) {
                        const uint32_t oa = ((kk >> 2) * (KT / 2) + (kk & 3) * 32) >> 4;
                        const uint32_t ob = ((kk >> 2) * (QT / 2) + (kk & 3) * 32) >> 4;
                        umma_ss(tmem + sb * 64, dk + oa, dq + ob, idesc_s, kk > 0);
                        umma_ss(tmem + (mode == 3 ? sb * 64 : 128 + sb * 64), dv + oa, dda + ob, idesc_s, 1);
                    }
                }
                if (mode != 1) {
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        const uint32_t ca = (kk >> 1) * 32 + (kk & 1) * 8;
                        umma_ts(tmem + 256, tmem + sb * 64 + ca, damn + kk * 128, idesc_a, 1);
                        umma_ts(tmem + 384, tmem + 128 + sb * 64 + ca, qmn + kk * 128, idesc_a, 1);
                    }
                }
            }
            __syncwarp();
        }
        if (elect_one()) umma_commit(&done);
        __syncwarp();
        mbar_wait(&done, 0);
        long long t1 = clock64();
        if (threadIdx.x == 32 && blockIdx.x == 0) out[0] = (t1 - t0) / steps;
    }
    tc_fence_before(); __syncthreads(); tc_fence_after();
    if (warp == 2) tmem_dealloc<512>(tmem);
}

int main() {
    long long* d; cudaMalloc(&d, 64);
    const int smem = 2 * KT + 2 * QT + 1024;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const char* names[] = {"full mix (16 SS N64 + 8 TS N128)", "SS part only", "TS part only", "SS part, one accumulator"};
    const int floor_[] = {1280, 768, 512, 768};
    for (int mode = 0; mode < 4; ++mode) {
        for (int rep = 0; rep < 2; ++rep) { k<<<148, 128, smem>>>(d, 2000, mode); cudaDeviceSynchronize(); }
        long long r; cudaMemcpy(&r, d, 8, cudaMemcpyDeviceToHost);
        printf("%-36s %5lld cyc/step (floor %d) %s\n", names[mode], r, floor_[mode], cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
