// tcgen05.mma kind::f16 issue throughput per SM (cycles per M=128,K=16 instruction) for
// A from SMEM (SS) or TMEM (TS), N in {32,64,128,256}, B K-major or MN-major, optionally with
// 8 warps streaming tcgen05.ld from TMEM at the same time (the attention epilogue's load).
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2602_16986_b200/csrc/sm100.cuh"
using namespace uh;

__global__ void __launch_bounds__(384, 1) k(float* out, int iters, int ts, int n, int bmn, int ldwarps, int ndst) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    __shared__ uint32_t slot;
    __shared__ __align__(8) uint64_t done;
    __shared__ volatile int stop;
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) ((uint32_t*)smem)[i] = 0;
    if (threadIdx.x == 0) { mbar_init(&done, 1); fence_barrier_init(); stop = 0; }
    if (warp == 2) tmem_alloc<512>(&slot);
    fence_proxy_async_smem();
    tc_fence_before(); __syncthreads(); tc_fence_after();
    const uint32_t tmem = slot;
    if (warp == 1) {
        long long t0 = clock64();
        if (elect_one()) {
            const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768);
            const uint32_t idesc = make_idesc_bf16(128, n, false, bmn != 0);
            uint64_t bd[4], ad[4];
            uint32_t dd[4];
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
                bd[kk] = bmn ? make_sw128_desc(b + kk * 2048, 8192, 1024) : make_sw128_desc(b + kk * 32, 16, 1024);
                ad[kk] = make_sw128_desc(a + kk * 32, 16, 1024);
                dd[kk] = tmem + (uint32_t)(kk % ndst) * (n < 64 ? 64 : n) % 256;
            }
            if (ts) {
                for (int i = 0; i < iters; i += 4) {
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) umma_ts(dd[kk], tmem + 256 + kk * 8, bd[kk], idesc, 1);
                }
            } else {
                for (int i = 0; i < iters; i += 4) {
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) umma_ss(dd[kk], ad[kk], bd[kk], idesc, 1);
                }
            }
            umma_commit(&done);
        }
        __syncwarp();
        mbar_wait(&done, 0);
        long long t1 = clock64();
        if (threadIdx.x == 32 && blockIdx.x == 0) out[0] = (float)(t1 - t0) / iters;
        stop = 1;
    } else if (warp >= 4 && warp - 4 < (ldwarps < 0 ? -ldwarps : ldwarps)) {
        const uint32_t base = tmem + ((uint32_t)((warp & 3) * 32) << 16) + 384 + ((warp - 4) >> 2) * 64;
        float v[32], acc = 0.f;
        long long cnt = 0;
        uint32_t wv[16];
        for (int i = 0; i < 16; ++i) wv[i] = i;
        while (!stop) {
            if (ldwarps > 0) { tmem_ld32(base, v); tmem_ld_wait(); acc += v[0]; }
            else { tmem_st16(base, wv); tmem_st_wait(); }
            ++cnt;
        }
        if (acc == 1.f) out[2] = acc;
        if (threadIdx.x == 128 && blockIdx.x == 0) out[1] = (float)cnt;
    }
    tc_fence_before(); __syncthreads(); tc_fence_after();
    if (warp == 2) tmem_dealloc<512>(tmem);
}

int main() {
    float* d; cudaMalloc(&d, 64);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
    const int iters = 40000;
    const int ndst = 1, bmn = 0;
    for (int ldw : {0, 4, 8, -4, -8})
        for (int ts = 0; ts < 2; ++ts)
                for (int n : {32, 128}) {
                    for (int rep = 0; rep < 2; ++rep) { k<<<148, 384, 80 * 1024>>>(d, iters, ts, n, bmn, ldw, ndst); cudaDeviceSynchronize(); }
                    float r[2]; cudaMemcpy(r, d, 8, cudaMemcpyDeviceToHost);
                    const double ldbw = (double)(ldw < 0 ? -ldw : ldw) * 32 * r[1] * (ldw < 0 ? 64 : 128) / (r[0] * iters);
                    const double floor = 128.0 * n / 256.0;
                    printf("ndst=%d %s B=%s N=%3d ldwarps=%d: %.2f cyc/mma (floor %.0f, %.0f%%)  ld-iters=%.0f tmem-%s %.0f B/clk %s\n",
                           ndst, ts ? "TS" : "SS", bmn ? "MN" : "K ", n, ldw, r[0], floor, 100.0 * floor / r[0], r[1], ldw < 0 ? "st" : "ld", ldbw,
                           cudaGetErrorString(cudaGetLastError()));
                }
    return 0;
}
