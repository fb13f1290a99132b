// tcgen05.mma issue cost and queue depth: bursts of B TS MMAs (M=128, K=16) into an idle tensor
// pipe; the issuing thread's clock around the burst (issue time) and around commit+wait (drain).
// Also the latency of mbarrier try_wait on an already-complete barrier, and of tcgen05.commit.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2602_16986_b200/csrc/sm100.cuh"
using namespace uh;

template <int B>
__device__ __forceinline__ void burst(uint32_t d, uint32_t a, uint64_t bd, uint32_t idesc) {
#pragma unroll
    for (int i = 0; i < B; ++i) umma_ts(d, a + (i & 3) * 8, bd + (i & 3) * 2, idesc, 1);
}

template <int B>
__global__ void __launch_bounds__(128, 1) k(long long* out, int n, int rounds) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    __shared__ uint32_t slot;
    __shared__ __align__(8) uint64_t done, dummy;
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 32 * 1024 / 4; i += blockDim.x) ((uint32_t*)smem)[i] = 0;
    if (threadIdx.x == 0) { mbar_init(&done, 1); mbar_init(&dummy, 1); fence_barrier_init(); }
    if (warp == 2) tmem_alloc<512>(&slot);
    fence_proxy_async_smem();
    tc_fence_before(); __syncthreads(); tc_fence_after();
    const uint32_t tmem = slot;
    if (warp == 1) {
        const uint32_t idesc = make_idesc_bf16(128, n, false, false);
        const uint64_t bd = make_sw128_desc(smem_u32(smem), 16, 1024);
        long long t_issue = 0, t_drain = 0, t_wait = 0, t_commit = 0;
        if (threadIdx.x == 32) { mbar_arrive(&dummy); }
        __syncwarp();
        for (int r = 0; r < rounds; ++r) {
            long long t0 = clock64();
            if (elect_one()) burst<B>(tmem, tmem + 256, bd, idesc);
            __syncwarp();
            long long t1 = clock64();
            if (elect_one()) umma_commit(&done);
            __syncwarp();
            long long t2 = clock64();
            mbar_wait(&done, r & 1);
            long long t3 = clock64();
            mbar_wait(&dummy, 0);   // already complete
            long long t4 = clock64();
            t_issue += t1 - t0; t_commit += t2 - t1; t_drain += t3 - t2; t_wait += t4 - t3;
        }
        if (threadIdx.x == 32 && blockIdx.x == 0) {
            out[0] = t_issue / rounds; out[1] = t_commit / rounds; out[2] = t_drain / rounds; out[3] = t_wait / rounds;
        }
    }
    tc_fence_before(); __syncthreads(); tc_fence_after();
    if (warp == 2) tmem_dealloc<512>(tmem);
}

template <int B>
void run(long long* d, int n) {
    cudaFuncSetAttribute(k<B>, cudaFuncAttributeMaxDynamicSharedMemorySize, 40 * 1024);
    for (int rep = 0; rep < 2; ++rep) { k<B><<<148, 128, 40 * 1024>>>(d, n, 200); cudaDeviceSynchronize(); }
    long long r[4]; cudaMemcpy(r, d, 32, cudaMemcpyDeviceToHost);
    printf("B=%2d N=%3d: issue %5lld cyc (%.1f/mma)  commit %lld  drain %5lld  (pipe work %d)  try_wait(done) %lld  %s\n",
           B, n, r[0], (double)r[0] / B, r[1], r[2], B * n / 2, r[3], cudaGetErrorString(cudaGetLastError()));
}

int main() {
    long long* d; cudaMalloc(&d, 64);
    for (int n : {32, 64, 128, 256}) { run<1>(d, n); run<4>(d, n); run<8>(d, n); run<16>(d, n); run<32>(d, n); run<64>(d, n); }
    return 0;
}
