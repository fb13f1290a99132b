// The attention forward's MMA-issuer loop in isolation: per tile 8 TS MMAs (N=64) + commit,
// then 4 TS MMAs (N=128) + commit, with two mbarrier waits per tile that are already complete
// (the data is "ready").  Variants: no waits; waits but no commits; test_wait instead of
// try_wait; waits hoisted (issued one block early).  Floor per tile: 512 cycles.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2602_16986_b200/csrc/sm100.cuh"
using namespace uh;

__device__ __forceinline__ bool mbar_test(uint32_t addr, uint32_t parity) {
    uint32_t ok;
    asm volatile("{\n\t.reg .pred P1;\n\tmbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n\tselp.b32 %0, 1, 0, P1;\n\t}"
                 : "=r"(ok) : "r"(addr), "r"(parity) : "memory");
    return ok != 0;
}

__global__ void __launch_bounds__(128, 1) k(long long* out, int tiles, int mode) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    __shared__ uint32_t slot;
    __shared__ __align__(8) uint64_t bars[8];
    __shared__ int flag;
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 32768 / 4; i += blockDim.x) ((uint32_t*)smem)[i] = 0;
    if (threadIdx.x == 0) {
        for (int i = 0; i < 8; ++i) mbar_init(&bars[i], 1);
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc<512>(&slot);
    fence_proxy_async_smem();
    tc_fence_before(); __syncthreads(); tc_fence_after();
    const uint32_t tmem = slot;
    if (warp == 1) {
        if (threadIdx.x == 32) { mbar_arrive(&bars[0]); mbar_arrive(&bars[1]); flag = 1 << 30; }   // "ready" 
        __syncwarp();
        constexpr uint32_t idesc_s = make_idesc_bf16(128, 64, false, false);
        constexpr uint32_t idesc_o = make_idesc_bf16(128, 128, false, true);
        const uint64_t kd = make_sw128_desc(smem_u32(smem), 16, 1024);
        const uint64_t vd = make_sw128_desc(smem_u32(smem) + 16384, 8192, 1024);
        const uint32_t a0 = smem_u32(&bars[0]), a1 = smem_u32(&bars[1]);
        long long t0 = clock64();
        if (mode == 8) {
            bool p0 = mbar_try_wait(a0, 0);
            for (int j = 0; j < tiles; ++j) {
                const int sb = j % 3;
                if (!p0) mbar_wait(&bars[0], 0);
                tc_fence_after();
                const bool p1 = mbar_try_wait(a1, 0);          // in flight while the S block issues
                if (elect_one()) {
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk)
                        umma_ts(tmem + sb * 64, tmem + 384 + kk * 8, kd + ((kk >> 2) * 8192 + (kk & 3) * 32) / 16, idesc_s, kk > 0);
                    umma_commit(&bars[2 + sb]);
                }
                __syncwarp();
                const int pb = (j + 1) % 3;
                if (!p1) mbar_wait(&bars[1], 0);
                tc_fence_after();
                p0 = mbar_try_wait(a0, 0);                     // in flight while the PV block issues
                if (elect_one()) {
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk)
                        umma_ts(tmem + 256, tmem + pb * 64 + (kk >> 1) * 32 + (kk & 1) * 8, vd + kk * 128, idesc_o, 1);
                    umma_commit(&bars[5]);
                }
                __syncwarp();
            }
        } else
        for (int j = 0; j < tiles; ++j) {
            const int sb = j % 3;
            if (mode == 6) { int v; do { asm volatile("ld.acquire.cta.shared::cta.b32 %0, [%1];" : "=r"(v) : "r"(smem_u32(&flag)) : "memory"); } while (v < j); }
            else if (mode == 7) { long long c0 = clock64(); while (clock64() - c0 < 150) { } }
            else if (mode != 1 && mode != 5) { if (mode == 3) { if (!mbar_test(a0, 0)) mbar_wait(&bars[0], 0); } else mbar_wait(&bars[0], 0); }
            if (mode != 4) tc_fence_after();
            if (elect_one()) {
#pragma unroll
                for (int kk = 0; kk < 8; ++kk)
                    umma_ts(tmem + sb * 64, tmem + 384 + kk * 8, kd + ((kk >> 2) * 8192 + (kk & 3) * 32) / 16, idesc_s, kk > 0);
                if (mode != 2) umma_commit(&bars[2 + sb]);
            }
            __syncwarp();
            const int pb = (j + 1) % 3;
            if (mode == 6) { int v; do { asm volatile("ld.acquire.cta.shared::cta.b32 %0, [%1];" : "=r"(v) : "r"(smem_u32(&flag)) : "memory"); } while (v < j); }
            else if (mode == 7) { long long c0 = clock64(); while (clock64() - c0 < 150) { } }
            else if (mode != 1 && mode != 5) { if (mode == 3) { if (!mbar_test(a1, 0)) mbar_wait(&bars[1], 0); } else mbar_wait(&bars[1], 0); }
            if (mode != 4) tc_fence_after();
            if (elect_one()) {
#pragma unroll
                for (int kk = 0; kk < 4; ++kk)
                    umma_ts(tmem + 256, tmem + pb * 64 + (kk >> 1) * 32 + (kk & 1) * 8, vd + kk * 128, idesc_o, 1);
                if (mode != 2) umma_commit(&bars[5]);
            }
            __syncwarp();
        }
        if (elect_one()) umma_commit(&bars[6]);
        __syncwarp();
        mbar_wait(&bars[6], 0);
        long long t1 = clock64();
        if (threadIdx.x == 32 && blockIdx.x == 0) out[0] = (t1 - t0) / tiles;
    }
    tc_fence_before(); __syncthreads(); tc_fence_after();
    if (warp == 2) tmem_dealloc<512>(tmem);
}

int main() {
    long long* d; cudaMalloc(&d, 64);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 40 * 1024);
    const char* names[] = {"waits + commits (kernel pattern)", "no waits", "waits, no commits", "test_wait fast path",
                           "waits, no tcgen05 fence", "fence, no waits", "flag poll (ld.acquire) + fence", "150-cycle busy delay + fence",
                           "try_wait issued one block early"};
    for (int mode = 0; mode < 9; ++mode) {
        for (int rep = 0; rep < 2; ++rep) { k<<<148, 128, 40 * 1024>>>(d, 2000, mode); cudaDeviceSynchronize(); }
        long long r; cudaMemcpy(&r, d, 8, cudaMemcpyDeviceToHost);
        printf("%-34s %5lld cyc/tile (floor 512) %s\n", names[mode], r, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
