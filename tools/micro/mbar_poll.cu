// mbarrier state word: which bit flips when a phase completes, and the latency of reading it
// with ld.acquire.shared versus mbarrier.try_wait on an already-complete phase.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2602_16986_b200/csrc/sm100.cuh"
using namespace uh;

__device__ __forceinline__ uint64_t ld_acq(uint32_t addr) {
    uint64_t v;
    asm volatile("ld.acquire.cta.shared::cta.b64 %0, [%1];" : "=l"(v) : "r"(addr) : "memory");
    return v;
}

__global__ void k(unsigned long long* out) {
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
    __syncthreads();
    if (threadIdx.x != 0) return;
    const uint32_t a = smem_u32(&bar);
    out[0] = ld_acq(a);                // fresh, phase 0 in progress
    mbar_arrive(&bar);
    out[1] = ld_acq(a);                // phase 0 complete
    mbar_arrive(&bar);
    out[2] = ld_acq(a);                // phase 1 complete
    // latencies (phase 0 and 1 complete; current phase 2 has parity 0)
    long long t0 = clock64();
    uint64_t acc = 0;
    for (int i = 0; i < 100; ++i) acc += ld_acq(a) >> 63;
    long long t1 = clock64();
    int ok = 0;
    for (int i = 0; i < 100; ++i) ok += mbar_try_wait(a, 1);
    long long t2 = clock64();
    out[3] = (t1 - t0) / 100;
    out[4] = (t2 - t1) / 100;
    out[5] = acc + ok;
}

int main() {
    unsigned long long* d; cudaMalloc(&d, 64);
    k<<<1, 32>>>(d);
    unsigned long long h[6]; cudaMemcpy(h, d, 48, cudaMemcpyDeviceToHost);
    printf("init %016llx\nafter phase0 %016llx\nafter phase1 %016llx\nld.acquire %llu cyc  try_wait(done) %llu cyc  (%llu) %s\n",
           h[0], h[1], h[2], h[3], h[4], h[5], cudaGetErrorString(cudaGetLastError()));
    return 0;
}
