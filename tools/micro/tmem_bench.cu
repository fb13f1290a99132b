// tcgen05.ld / tcgen05.st throughput per SM (bytes per clock), 4..12 warps reading/writing TMEM.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2602_16986_b200/csrc/sm100.cuh"
using namespace uh;

template <int MODE>
__global__ void __launch_bounds__(512, 1) k(float* out, int iters, int nwarps) {
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) tmem_alloc<512>(&slot);
    tc_fence_before(); __syncthreads(); tc_fence_after();
    const uint32_t tmem = slot;
    float acc = 0.f;
    long long t0 = clock64();
    if (warp < nwarps) {
        const uint32_t base = tmem + ((uint32_t)((warp & 3) * 32) << 16) + (warp >> 2) * 64;
        float v[32];
        uint32_t w[16];
        for (int i = 0; i < 16; ++i) w[i] = i;
        for (int it = 0; it < iters; ++it) {
            if (MODE == 0) {
                tmem_ld32(base + (it & 1) * 32, v);
                tmem_ld_wait();
                acc += v[0] + v[31];
            } else {
                tmem_st16(base + (it & 3) * 16, w);
                tmem_st_wait();
            }
        }
    }
    long long t1 = clock64();
    __syncthreads();
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (float)(t1 - t0);
    if (acc == 123.f) out[1] = acc;
    if (warp == 0) tmem_dealloc<512>(tmem);
}

int main() {
    float* d; cudaMalloc(&d, 64);
    const int iters = 20000;
    for (int mode = 0; mode < 2; ++mode)
        for (int nw : {4, 8, 12, 16}) {
            for (int rep = 0; rep < 2; ++rep) {
                if (mode == 0) k<0><<<148, 512>>>(d, iters, nw); else k<1><<<148, 512>>>(d, iters, nw);
                cudaDeviceSynchronize();
            }
            float cyc; cudaMemcpy(&cyc, d, 4, cudaMemcpyDeviceToHost);
            double bytes = (double)nw * 32 * iters * (mode == 0 ? 32 * 4 : 16 * 4);
            printf("%s warps=%2d  %.1f B/clk/SM  (%.0f cycles)  err=%s\n", mode == 0 ? "ld.32x32b.x32" : "st.32x32b.x16",
                   nw, bytes / cyc, cyc, cudaGetErrorString(cudaGetLastError()));
        }
    return 0;
}
