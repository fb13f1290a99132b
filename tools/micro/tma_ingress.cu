// Global -> shared ingress per SM with cp.async.bulk (the TMA bulk path): every CTA streams
// CHUNK-byte pieces of a buffer through a 4-deep shared ring.  Source sizes: L2-resident
// (16 MB, every SM reads the same region) and HBM (2 GB, disjoint slices).  Bytes/clk/SM.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2602_16986_b200/csrc/sm100.cuh"
using namespace uh;


__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

template <int CHUNK, int DEPTH>
__global__ void __launch_bounds__(64, 1) k(const uint8_t* src, size_t span, int iters, long long* out, int shared_src) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ __align__(8) uint64_t full[DEPTH];
    if (threadIdx.x == 0) { for (int i = 0; i < DEPTH; ++i) mbar_init(&full[i], 1); fence_barrier_init(); }
    __syncthreads();
    if (threadIdx.x != 0) return;
    const uint8_t* base = shared_src ? src : src + (size_t)blockIdx.x * span;
    const size_t nchunks = span / CHUNK;
    long long t0 = clock64();
    for (int i = 0; i < iters + DEPTH; ++i) {
        if (i >= DEPTH) mbar_wait(&full[i % DEPTH], ((i / DEPTH) - 1) & 1);
        if (i < iters) {
            mbar_arrive_expect_tx(&full[i % DEPTH], CHUNK);
            bulk_g2s(smem + (i % DEPTH) * CHUNK, base + ((size_t)(i + blockIdx.x * 7) % nchunks) * CHUNK, CHUNK, &full[i % DEPTH]);
        }
    }
    long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = t1 - t0;
}

template <int CHUNK, int DEPTH>
void run(const uint8_t* d, size_t bytes, long long* o, int shared_src, const char* name) {
    cudaFuncSetAttribute(k<CHUNK, DEPTH>, cudaFuncAttributeMaxDynamicSharedMemorySize, DEPTH * CHUNK);
    const int iters = 2000;
    const size_t span = shared_src ? (16u << 20) : (bytes / 148) & ~(size_t)65535;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    k<CHUNK, DEPTH><<<148, 64, DEPTH * CHUNK>>>(d, span, 10, o, shared_src);
    cudaEventRecord(e0);
    k<CHUNK, DEPTH><<<148, 64, DEPTH * CHUNK>>>(d, span, iters, o, shared_src);
    cudaEventRecord(e1);
    cudaDeviceSynchronize();
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    long long cyc; cudaMemcpy(&cyc, o, 8, cudaMemcpyDeviceToHost);
    const double tot = 148.0 * iters * CHUNK;
    printf("%-10s depth %d chunk %6d B: %6.1f B/clk/SM (%.0f cycles), chip %.2f TB/s  %s\n", name, DEPTH, CHUNK, (double)iters * CHUNK / cyc,
           (double)cyc, tot / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    const size_t bytes = (size_t)2 << 30;
    uint8_t* d; cudaMalloc(&d, bytes); cudaMemset(d, 1, bytes);
    long long* o; cudaMalloc(&o, 64);
    for (int s = 1; s >= 0; --s) {
        const char* nm = s ? "L2 (16MB)" : "HBM (2GB)";
        run<16384, 4>(d, bytes, o, s, nm);
        run<32768, 4>(d, bytes, o, s, nm);
        run<16384, 8>(d, bytes, o, s, nm);
        run<32768, 6>(d, bytes, o, s, nm);
    }
    return 0;
}
