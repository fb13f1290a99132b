// Throughput of the SFU (MUFU) functions the SiLU epilogues can use, per SM per clock.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

template <int OP>
__global__ void k(float* out, int iters) {
    float x0 = threadIdx.x * 1e-3f, x1 = x0 + 0.1f, x2 = x0 + 0.2f, x3 = x0 + 0.3f;
    float x4 = x0 + 0.4f, x5 = x0 + 0.5f, x6 = x0 + 0.6f, x7 = x0 + 0.7f;
    uint32_t p0 = 0x3e803e80u + threadIdx.x, p1 = p0 + 1, p2 = p0 + 2, p3 = p0 + 3;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#define F1(x) if (OP == 0) asm volatile("tanh.approx.f32 %0, %0;" : "+f"(x)); \
              else if (OP == 1) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x)); \
              else if (OP == 2) asm volatile("rcp.approx.ftz.f32 %0, %0;" : "+f"(x));
        if (OP <= 2) { F1(x0) F1(x1) F1(x2) F1(x3) F1(x4) F1(x5) F1(x6) F1(x7) }
        if (OP == 3) {
            asm volatile("tanh.approx.bf16x2 %0, %0;" : "+r"(p0)); asm volatile("tanh.approx.bf16x2 %0, %0;" : "+r"(p1));
            asm volatile("tanh.approx.bf16x2 %0, %0;" : "+r"(p2)); asm volatile("tanh.approx.bf16x2 %0, %0;" : "+r"(p3));
        }
        if (OP == 4) {
            asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(p0)); asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(p1));
            asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(p2)); asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(p3));
        }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) out[1] = (float)(t1 - t0);
    out[2 + threadIdx.x % 8] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7 + __uint_as_float(p0 ^ p1 ^ p2 ^ p3);
}

int main() {
    float* d; cudaMalloc(&d, 1024);
    const char* names[] = {"tanh.f32", "ex2.f32", "rcp.f32", "tanh.bf16x2", "ex2.bf16x2"};
    const int iters = 4096, threads = 512, blocks = 148;
    for (int op = 0; op < 5; ++op) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
            cudaEventRecord(e0);
            switch (op) {
                case 0: k<0><<<blocks, threads>>>(d, iters); break;
                case 1: k<1><<<blocks, threads>>>(d, iters); break;
                case 2: k<2><<<blocks, threads>>>(d, iters); break;
                case 3: k<3><<<blocks, threads>>>(d, iters); break;
                default: k<4><<<blocks, threads>>>(d, iters); break;
            }
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            float cyc; cudaMemcpy(&cyc, d + 1, 4, cudaMemcpyDeviceToHost);
            double ops_per_sm = (double)threads * iters * (op <= 2 ? 8 : 8);  // elements (bf16x2: 4 ops x 2 elements)
            if (rep) printf("%-12s %8.3f ms  %6.2f elements/clk/SM (clock64-based)\n", names[op], ms, ops_per_sm / cyc);
        }
    }
    return 0;
}
