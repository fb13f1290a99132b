// norm.cu — HBM-bound row kernels of the layer: input LayerNorm (Eq. 1),
// gated norm Y = Norm(A) (.) U (Eq. 4; "fused gated normalization kernel"
// P:187) and their backward passes, the x^ rematerialisation from saved statistics
// ("reusing saved layer-norm statistics") and column sums.
//
// One warp per row, 16-byte vector accesses (8 bf16 or 4 fp32 per access),
// coalesced along the row; parameter-gradient partial sums are held in registers
// across a grid-stride loop over rows and reduced once per block.
#include <cuda_bf16.h>

#include <algorithm>
#include <initializer_list>
#include <utility>

#include "internal.h"
#include "sm100.cuh"

namespace uh {
namespace {

template <typename T> struct Vec;
template <> struct Vec<float> {
    static constexpr int N = 4;
    __device__ __forceinline__ static void load(const float* p, float* v) {
        float4 a = *reinterpret_cast<const float4*>(p);
        v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
    }
    __device__ __forceinline__ static void store(float* p, const float* v) {
        *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
    }
};
template <> struct Vec<__nv_bfloat16> {
    static constexpr int N = 8;
    __device__ __forceinline__ static void load(const __nv_bfloat16* p, float* v) {
        uint4 a = *reinterpret_cast<const uint4*>(p);
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&a);
#pragma unroll
        for (int i = 0; i < 4; ++i) { float2 f = __bfloat1622float2(h[i]); v[2 * i] = f.x; v[2 * i + 1] = f.y; }
    }
    __device__ __forceinline__ static void store(__nv_bfloat16* p, const float* v) {
        uint4 a;
        __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&a);
#pragma unroll
        for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
        *reinterpret_cast<uint4*>(p) = a;
    }
};
__device__ __forceinline__ void load4f(const float* p, float* v) { Vec<float>::load(p, v); }

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

constexpr int kRowsPerBlock = 8;  // 8 warps

// ------------------------------------------------------------------ LN forward
template <typename T, int CPL>
__global__ void __launch_bounds__(256) ln_fwd_k(int64_t nrows, int d, const T* __restrict__ x, int64_t ldx,
                                                const float* __restrict__ w, const float* __restrict__ b, float eps,
                                                T* __restrict__ y, int64_t ldy, float* mean, float* rstd) {
    constexpr int V = Vec<T>::N;
    const int lane = threadIdx.x & 31;
    const int64_t row = (int64_t)blockIdx.x * kRowsPerBlock + (threadIdx.x >> 5);
    if (row >= nrows) return;
    const int nch = d / V;
    float v[CPL][V];
    float s = 0.f;
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
        int ch = lane + 32 * c;
        if (ch < nch) {
            Vec<T>::load(x + row * ldx + ch * V, v[c]);
#pragma unroll
            for (int e = 0; e < V; ++e) s += v[c][e];
        }
    }
    const float mu = warp_sum(s) / d;
    float q = 0.f;
#pragma unroll
    for (int c = 0; c < CPL; ++c)
        if (lane + 32 * c < nch)
#pragma unroll
            for (int e = 0; e < V; ++e) { float t = v[c][e] - mu; q += t * t; }
    const float rs = rsqrtf(warp_sum(q) / d + eps);
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
        int ch = lane + 32 * c;
        if (ch < nch) {
            float wv[V], bv[V], o[V];
#pragma unroll
            for (int e = 0; e < V; e += 4) { load4f(w + ch * V + e, wv + e); load4f(b + ch * V + e, bv + e); }
#pragma unroll
            for (int e = 0; e < V; ++e) o[e] = (v[c][e] - mu) * rs * wv[e] + bv[e];
            Vec<T>::store(y + row * ldy + ch * V, o);
        }
    }
    if (lane == 0) {
        if (mean) mean[row] = mu;
        if (rstd) rstd[row] = rs;
    }
}

template <typename T, int CPL>
__global__ void __launch_bounds__(256) ln_apply_k(int64_t nrows, int d, const T* __restrict__ x, int64_t ldx,
                                                  const float* __restrict__ w, const float* __restrict__ b,
                                                  const float* __restrict__ mean, const float* __restrict__ rstd,
                                                  T* __restrict__ y, int64_t ldy) {
    constexpr int V = Vec<T>::N;
    const int lane = threadIdx.x & 31;
    const int64_t row = (int64_t)blockIdx.x * kRowsPerBlock + (threadIdx.x >> 5);
    if (row >= nrows) return;
    const int nch = d / V;
    const float mu = mean[row], rs = rstd[row];
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
        int ch = lane + 32 * c;
        if (ch < nch) {
            float v[V], wv[V], bv[V];
            Vec<T>::load(x + row * ldx + ch * V, v);
#pragma unroll
            for (int e = 0; e < V; e += 4) { load4f(w + ch * V + e, wv + e); load4f(b + ch * V + e, bv + e); }
#pragma unroll
            for (int e = 0; e < V; ++e) v[e] = (v[e] - mu) * rs * wv[e] + bv[e];
            Vec<T>::store(y + row * ldy + ch * V, v);
        }
    }
}

// ------------------------------------------------------------------ gated norm forward
template <typename T, int CPL>
__global__ void __launch_bounds__(256) gated_fwd_k(int64_t nrows, int d, const T* __restrict__ A, int64_t lda,
                                                   const T* __restrict__ U, int64_t ldu, const float* __restrict__ w,
                                                   const float* __restrict__ b, float eps, T* __restrict__ Y,
                                                   int64_t ldy, float* mean, float* rstd) {
    constexpr int V = Vec<T>::N;
    const int lane = threadIdx.x & 31;
    const int64_t row = (int64_t)blockIdx.x * kRowsPerBlock + (threadIdx.x >> 5);
    if (row >= nrows) return;
    const int nch = d / V;
    float v[CPL][V];
    float s = 0.f;
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
        int ch = lane + 32 * c;
        if (ch < nch) {
            Vec<T>::load(A + row * lda + ch * V, v[c]);
#pragma unroll
            for (int e = 0; e < V; ++e) s += v[c][e];
        }
    }
    const float mu = warp_sum(s) / d;
    float q = 0.f;
#pragma unroll
    for (int c = 0; c < CPL; ++c)
        if (lane + 32 * c < nch)
#pragma unroll
            for (int e = 0; e < V; ++e) { float t = v[c][e] - mu; q += t * t; }
    const float rs = rsqrtf(warp_sum(q) / d + eps);
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
        int ch = lane + 32 * c;
        if (ch < nch) {
            float wv[V], bv[V], u[V], o[V];
            Vec<T>::load(U + row * ldu + ch * V, u);
#pragma unroll
            for (int e = 0; e < V; e += 4) { load4f(w + ch * V + e, wv + e); load4f(b + ch * V + e, bv + e); }
#pragma unroll
            for (int e = 0; e < V; ++e) o[e] = ((v[c][e] - mu) * rs * wv[e] + bv[e]) * u[e];
            Vec<T>::store(Y + row * ldy + ch * V, o);
        }
    }
    if (lane == 0) {
        if (mean) mean[row] = mu;
        if (rstd) rstd[row] = rs;
    }
}

// ------------------------------------------------------------------ NEXT-2: norms fused with row-wise E4M3
// quantisation (Fig. fp8: "fuse the scaling/quantization steps with the preceding kernels").
// The row's normalised values stay in registers (fp32); amax by warp max; s = amax / 448,
// code = E4M3_rn_sat(v * (448 / amax)) in fp32 (readings R18, R19); an all-zero row gets s = 1.
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

template <int CPL>
__device__ __forceinline__ void quant_row_store(float (&o)[CPL][8], int lane, int nch, uint8_t* q, float* scale,
                                                int64_t row) {
    float am = 0.f;
#pragma unroll
    for (int c = 0; c < CPL; ++c)
        if (lane + 32 * c < nch)
#pragma unroll
            for (int e = 0; e < 8; ++e) am = fmaxf(am, fabsf(o[c][e]));
    am = warp_max(am);
    const float inv = am > 0.f ? __fdiv_rn(448.f, am) : 1.f;
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
        const int ch = lane + 32 * c;
        if (ch < nch) {
            uint2 pk;
            pk.x = (uint32_t)cvt_e4m3x2(__fmul_rn(o[c][0], inv), __fmul_rn(o[c][1], inv))
                 | ((uint32_t)cvt_e4m3x2(__fmul_rn(o[c][2], inv), __fmul_rn(o[c][3], inv)) << 16);
            pk.y = (uint32_t)cvt_e4m3x2(__fmul_rn(o[c][4], inv), __fmul_rn(o[c][5], inv))
                 | ((uint32_t)cvt_e4m3x2(__fmul_rn(o[c][6], inv), __fmul_rn(o[c][7], inv)) << 16);
            *reinterpret_cast<uint2*>(q + ch * 8) = pk;
        }
    }
    if (lane == 0) scale[row] = am > 0.f ? __fdiv_rn(am, 448.f) : 1.f;
}

template <int CPL>
__global__ void __launch_bounds__(256) ln_fwd_fp8_k(int64_t nrows, int d, const __nv_bfloat16* __restrict__ x,
                                                    int64_t ldx, const float* __restrict__ w,
                                                    const float* __restrict__ b, float eps, uint8_t* __restrict__ q,
                                                    int64_t ldq, float* __restrict__ scale, float* mean, float* rstd) {
    const int lane = threadIdx.x & 31;
    const int64_t row = (int64_t)blockIdx.x * kRowsPerBlock + (threadIdx.x >> 5);
    if (row >= nrows) return;
    const int nch = d / 8;
    float v[CPL][8];
    float s = 0.f;
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
        const int ch = lane + 32 * c;
        if (ch < nch) {
            Vec<__nv_bfloat16>::load(x + row * ldx + ch * 8, v[c]);
#pragma unroll
            for (int e = 0; e < 8; ++e) s += v[c][e];
        }
    }
    const float mu = warp_sum(s) / d;
    float qq = 0.f;
#pragma unroll
    for (int c = 0; c < CPL; ++c)
        if (lane + 32 * c < nch)
#pragma unroll
            for (int e = 0; e < 8; ++e) { float t = v[c][e] - mu; qq += t * t; }
    const float rs = rsqrtf(warp_sum(qq) / d + eps);
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
        const int ch = lane + 32 * c;
        if (ch < nch) {
            float wv[8], bv[8];
            load4f(w + ch * 8, wv); load4f(w + ch * 8 + 4, wv + 4);
            load4f(b + ch * 8, bv); load4f(b + ch * 8 + 4, bv + 4);
#pragma unroll
            for (int e = 0; e < 8; ++e) v[c][e] = (v[c][e] - mu) * rs * wv[e] + bv[e];
        }
    }
    quant_row_store<CPL>(v, lane, nch, q + row * ldq, scale, row);
    if (lane == 0) {
        if (mean) mean[row] = mu;
        if (rstd) rstd[row] = rs;
    }
}

template <int CPL>
__global__ void __launch_bounds__(256) gated_fwd_fp8_k(int64_t nrows, int d, const __nv_bfloat16* __restrict__ A,
                                                       int64_t lda, const __nv_bfloat16* __restrict__ U, int64_t ldu,
                                                       const float* __restrict__ w, const float* __restrict__ b,
                                                       float eps, uint8_t* __restrict__ q, int64_t ldq,
                                                       float* __restrict__ scale, float* mean, float* rstd) {
    const int lane = threadIdx.x & 31;
    const int64_t row = (int64_t)blockIdx.x * kRowsPerBlock + (threadIdx.x >> 5);
    if (row >= nrows) return;
    const int nch = d / 8;
    float v[CPL][8], u[CPL][8];
    float s = 0.f;
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
        const int ch = lane + 32 * c;
        if (ch < nch) {
            Vec<__nv_bfloat16>::load(A + row * lda + ch * 8, v[c]);
            Vec<__nv_bfloat16>::load(U + row * ldu + ch * 8, u[c]);
#pragma unroll
            for (int e = 0; e < 8; ++e) s += v[c][e];
        }
    }
    const float mu = warp_sum(s) / d;
    float qq = 0.f;
#pragma unroll
    for (int c = 0; c < CPL; ++c)
        if (lane + 32 * c < nch)
#pragma unroll
            for (int e = 0; e < 8; ++e) { float t = v[c][e] - mu; qq += t * t; }
    const float rs = rsqrtf(warp_sum(qq) / d + eps);
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
        const int ch = lane + 32 * c;
        if (ch < nch) {
            float wv[8], bv[8];
            load4f(w + ch * 8, wv); load4f(w + ch * 8 + 4, wv + 4);
            load4f(b + ch * 8, bv); load4f(b + ch * 8 + 4, bv + 4);
#pragma unroll
            for (int e = 0; e < 8; ++e) v[c][e] = ((v[c][e] - mu) * rs * wv[e] + bv[e]) * u[c][e];
        }
    }
    quant_row_store<CPL>(v, lane, nch, q + row * ldq, scale, row);
    if (lane == 0) {
        if (mean) mean[row] = mu;
        if (rstd) rstd[row] = rs;
    }
}

// weight W [K, N] (bf16, row stride ldw) -> W^T codes [N, K] (K-major, row stride ldq bytes) and one scale
// per output column (R18).  Block = 32 columns x 8 row groups; the transposed codes are written
// through a shared-memory tile so both the reads and the writes are coalesced.
__global__ void __launch_bounds__(256) quant_weight_fp8_k(int K, int N, const __nv_bfloat16* __restrict__ W,
                                                          int64_t ldw, uint8_t* __restrict__ qt, int64_t ldq,
                                                          float* __restrict__ scale) {
    __shared__ float red[8][33];
    __shared__ uint8_t tile[32][33];
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const int n = blockIdx.x * 32 + tx;
    float am = 0.f;
    if (n < N)
        for (int k = ty; k < K; k += 8) am = fmaxf(am, fabsf(__bfloat162float(W[(int64_t)k * ldw + n])));
    red[ty][tx] = am;
    __syncthreads();
    if (ty == 0) {
        for (int i = 1; i < 8; ++i) am = fmaxf(am, red[i][tx]);
        red[0][tx] = am;
        if (n < N) scale[n] = am > 0.f ? __fdiv_rn(am, 448.f) : 1.f;
    }
    __syncthreads();
    const float colmax = red[0][tx];
    const float inv = colmax > 0.f ? __fdiv_rn(448.f, colmax) : 1.f;
    for (int k0 = 0; k0 < K; k0 += 32) {
        for (int kk = ty; kk < 32; kk += 8) {   // read rows k0 + kk, column n
            const int k = k0 + kk;
            const float v = (n < N && k < K) ? __bfloat162float(W[(int64_t)k * ldw + n]) : 0.f;
            tile[tx][kk] = (uint8_t)(cvt_e4m3x2(__fmul_rn(v, inv), 0.f) & 0xFF);
        }
        __syncthreads();
        for (int nn = ty; nn < 32; nn += 8) {   // write qt[n0 + nn][k0 + tx]
            const int n2 = blockIdx.x * 32 + nn, k = k0 + tx;
            if (n2 < N && k < K) qt[(int64_t)n2 * ldq + k] = tile[nn][tx];
        }
        __syncthreads();
    }
}

// block-level reduction of per-lane parameter-gradient partials, then one atomic per column
template <typename T, int CPL>
__device__ __forceinline__ void flush_param_grads(int d, float (*pw)[Vec<T>::N], float (*pb)[Vec<T>::N], float* dw,
                                                  float* db, float* red /* smem [2][d] */) {
    constexpr int V = Vec<T>::N;
    const int lane = threadIdx.x & 31;
    const int nch = d / V;
    for (int i = threadIdx.x; i < 2 * d; i += blockDim.x) red[i] = 0.f;
    __syncthreads();
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
        int ch = lane + 32 * c;
        if (ch < nch)
#pragma unroll
            for (int e = 0; e < V; ++e) {
                atomicAdd(&red[ch * V + e], pw[c][e]);
                atomicAdd(&red[d + ch * V + e], pb[c][e]);
            }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < d; i += blockDim.x) {
        if (dw) atomicAdd(dw + i, red[i]);
        if (db) atomicAdd(db + i, red[d + i]);
    }
}

// ------------------------------------------------------------------ gated norm backward
// Given dY: A^ = (A - mu) rstd w + b, Y = A^ U;  dA^ = dY U, dU = dY A^ -> dH_U = dU * G_U;
// dA = rstd (g - mean(g) - x~ mean(g x~)), g = dA^ w;  dw += dA^ x~, db += dA^.
template <typename T, int CPL>
__global__ void __launch_bounds__(256) gated_bwd_k(int64_t nrows, int d, const T* __restrict__ dY, int64_t lddy,
                                                   const T* __restrict__ A, int64_t lda, const T* __restrict__ U,
                                                   int64_t ldu, const T* __restrict__ GU, int64_t ldg,
                                                   const float* __restrict__ w, const float* __restrict__ b,
                                                   const float* __restrict__ mean, const float* __restrict__ rstd,
                                                   T* __restrict__ dA, int64_t ldda, T* __restrict__ dHU, int64_t ldh,
                                                   T* __restrict__ Y, int64_t ldy, float* dw, float* db) {
    constexpr int V = Vec<T>::N;
    extern __shared__ float red[];
    const int lane = threadIdx.x & 31;
    const int nch = d / V;
    float pw[CPL][V], pb[CPL][V];
#pragma unroll
    for (int c = 0; c < CPL; ++c)
#pragma unroll
        for (int e = 0; e < V; ++e) { pw[c][e] = 0.f; pb[c][e] = 0.f; }
    for (int64_t row = (int64_t)blockIdx.x * kRowsPerBlock + (threadIdx.x >> 5); row < nrows;
         row += (int64_t)gridDim.x * kRowsPerBlock) {
        const float mu = mean[row], rs = rstd[row];
        float xt[CPL][V], g[CPL][V];
        float sg = 0.f, sgx = 0.f;
#pragma unroll
        for (int c = 0; c < CPL; ++c) {
            int ch = lane + 32 * c;
            if (ch < nch) {
                float a[V], u[V], dy[V], gu[V], wv[V], bv[V], y[V], dh[V];
                Vec<T>::load(A + row * lda + ch * V, a);
                Vec<T>::load(U + row * ldu + ch * V, u);
                Vec<T>::load(dY + row * lddy + ch * V, dy);
                Vec<T>::load(GU + row * ldg + ch * V, gu);
#pragma unroll
                for (int e = 0; e < V; e += 4) { load4f(w + ch * V + e, wv + e); load4f(b + ch * V + e, bv + e); }
#pragma unroll
                for (int e = 0; e < V; ++e) {
                    xt[c][e] = (a[e] - mu) * rs;
                    float ah = xt[c][e] * wv[e] + bv[e];
                    y[e] = ah * u[e];
                    float dah = dy[e] * u[e];
                    dh[e] = dy[e] * ah * gu[e];
                    g[c][e] = dah * wv[e];
                    pw[c][e] += dah * xt[c][e];
                    pb[c][e] += dah;
                    sg += g[c][e];
                    sgx += g[c][e] * xt[c][e];
                }
                if (Y) Vec<T>::store(Y + row * ldy + ch * V, y);
                Vec<T>::store(dHU + row * ldh + ch * V, dh);
            }
        }
        const float mg = warp_sum(sg) / d, mgx = warp_sum(sgx) / d;
#pragma unroll
        for (int c = 0; c < CPL; ++c) {
            int ch = lane + 32 * c;
            if (ch < nch) {
                float o[V];
#pragma unroll
                for (int e = 0; e < V; ++e) o[e] = rs * (g[c][e] - mg - xt[c][e] * mgx);
                Vec<T>::store(dA + row * ldda + ch * V, o);
            }
        }
    }
    flush_param_grads<T, CPL>(d, pw, pb, dw, db, red);
}

// ------------------------------------------------------------------ LN backward (+ residual)
template <typename T, int CPL>
__global__ void __launch_bounds__(256) ln_bwd_k(int64_t nrows, int d, const T* __restrict__ dxh, int64_t ldg,
                                                const T* __restrict__ x, int64_t ldx, const float* __restrict__ w,
                                                const float* __restrict__ mean, const float* __restrict__ rstd,
                                                const T* __restrict__ dres, int64_t ldr, T* __restrict__ dx,
                                                int64_t lddx, float* dw, float* db) {
    constexpr int V = Vec<T>::N;
    extern __shared__ float red[];
    const int lane = threadIdx.x & 31;
    const int nch = d / V;
    float pw[CPL][V], pb[CPL][V];
#pragma unroll
    for (int c = 0; c < CPL; ++c)
#pragma unroll
        for (int e = 0; e < V; ++e) { pw[c][e] = 0.f; pb[c][e] = 0.f; }
    for (int64_t row = (int64_t)blockIdx.x * kRowsPerBlock + (threadIdx.x >> 5); row < nrows;
         row += (int64_t)gridDim.x * kRowsPerBlock) {
        const float mu = mean[row], rs = rstd[row];
        float xt[CPL][V], g[CPL][V], rr[CPL][V];
        float sg = 0.f, sgx = 0.f;
#pragma unroll
        for (int c = 0; c < CPL; ++c) {
            int ch = lane + 32 * c;
            if (ch < nch) {
                float xv[V], gv[V], wv[V];
                Vec<T>::load(x + row * ldx + ch * V, xv);
                Vec<T>::load(dxh + row * ldg + ch * V, gv);
                if (dres) Vec<T>::load(dres + row * ldr + ch * V, rr[c]);   // in flight with x, dx^
#pragma unroll
                for (int e = 0; e < V; e += 4) load4f(w + ch * V + e, wv + e);
#pragma unroll
                for (int e = 0; e < V; ++e) {
                    xt[c][e] = (xv[e] - mu) * rs;
                    g[c][e] = gv[e] * wv[e];
                    pw[c][e] += gv[e] * xt[c][e];
                    pb[c][e] += gv[e];
                    sg += g[c][e];
                    sgx += g[c][e] * xt[c][e];
                }
            }
        }
        const float mg = warp_sum(sg) / d, mgx = warp_sum(sgx) / d;
#pragma unroll
        for (int c = 0; c < CPL; ++c) {
            int ch = lane + 32 * c;
            if (ch < nch) {
                float o[V];
#pragma unroll
                for (int e = 0; e < V; ++e) o[e] = rs * (g[c][e] - mg - xt[c][e] * mgx) + (dres ? rr[c][e] : 0.f);
                Vec<T>::store(dx + row * lddx + ch * V, o);
            }
        }
    }
    flush_param_grads<T, CPL>(d, pw, pb, dw, db, red);
}

// ------------------------------------------------------------------ pipelined backward rows (bf16)
// The same arithmetic as gated_bwd_k / ln_bwd_k with the rows' inputs streamed into a per-warp
// shared-memory ring by cp.async.bulk (one lane issues, DEPTH rows ahead): 16 warps per SM
// keep DEPTH x NT KB in flight each instead of one row, enough to cover HBM latency.
constexpr int kPipeWarps = 8;

template <int NT, int DEPTH>
struct RowRing {
    uint8_t* buf;   // this warp's [DEPTH][NT][row bytes]
    uint64_t* bar;  // [DEPTH]
    int rb;
    __device__ __forceinline__ const uint8_t* slot(int s, int t) const { return buf + (s * NT + t) * rb; }
    // lane 0: fill slot s with row `row` of the NT sources
    __device__ __forceinline__ void issue(int s, const uint8_t* const* src, const int64_t* ld_bytes, int64_t row) {
        fence_proxy_async_smem();   // the warp's generic reads of this slot (synced) precede the async writes
        mbar_arrive_expect_tx(&bar[s], (uint32_t)(NT * rb));
#pragma unroll
        for (int t = 0; t < NT; ++t) bulk_load_1d(buf + (s * NT + t) * rb, src[t] + row * ld_bytes[t], rb, &bar[s]);
    }
};

__device__ __forceinline__ void bf16x8_to_f32(uint4 a, float* v) {
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&a);
#pragma unroll
    for (int i = 0; i < 4; ++i) { float2 f = __bfloat1622float2(h[i]); v[2 * i] = f.x; v[2 * i + 1] = f.y; }
}

template <int CPL, int DEPTH>
__global__ void __launch_bounds__(256) gated_bwd_pipe_k(int64_t nrows, int d, const __nv_bfloat16* __restrict__ dY,
                                                        int64_t lddy, const __nv_bfloat16* __restrict__ A, int64_t lda,
                                                        const __nv_bfloat16* __restrict__ U, int64_t ldu,
                                                        const __nv_bfloat16* __restrict__ GU, int64_t ldg,
                                                        const float* __restrict__ w, const float* __restrict__ b,
                                                        const float* __restrict__ mean, const float* __restrict__ rstd,
                                                        __nv_bfloat16* __restrict__ dA, int64_t ldda,
                                                        __nv_bfloat16* __restrict__ dHU, int64_t ldh,
                                                        __nv_bfloat16* __restrict__ Y, int64_t ldy, float* dw, float* db) {
    using T = __nv_bfloat16;
    constexpr int V = 8, NT = 4;
    extern __shared__ __align__(128) uint8_t pipe_smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int rb = d * 2, nch = d / V;
    float* red = reinterpret_cast<float*>(pipe_smem);                     // [2][d] (flush_param_grads)
    uint64_t* bars = reinterpret_cast<uint64_t*>(pipe_smem + 2 * d * 4);  // [8 warps][DEPTH]
    uint8_t* ring0 = pipe_smem + 2 * d * 4 + kPipeWarps * DEPTH * 8;
    ring0 += (128 - (reinterpret_cast<uintptr_t>(ring0) & 127)) & 127;
    RowRing<NT, DEPTH> rr{ring0 + (size_t)warp * DEPTH * NT * rb, bars + warp * DEPTH, rb};
    const uint8_t* src[NT] = {reinterpret_cast<const uint8_t*>(A), reinterpret_cast<const uint8_t*>(U),
                              reinterpret_cast<const uint8_t*>(dY), reinterpret_cast<const uint8_t*>(GU)};
    const int64_t ldb[NT] = {lda * 2, ldu * 2, lddy * 2, ldg * 2};
    const int64_t G = (int64_t)gridDim.x * kPipeWarps;
    const int64_t r0 = (int64_t)blockIdx.x * kPipeWarps + warp;
    if (lane == 0) {
        for (int s = 0; s < DEPTH; ++s) mbar_init(&rr.bar[s], 1);
        fence_barrier_init();
        for (int s = 0; s < DEPTH; ++s)
            if (r0 + s * G < nrows) rr.issue(s, src, ldb, r0 + s * G);
    }
    __syncwarp();
    float wv[CPL][V], bv[CPL][V], pw[CPL][V], pb[CPL][V];
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
        const int ch = lane + 32 * c;
#pragma unroll
        for (int e = 0; e < V; ++e) { pw[c][e] = 0.f; pb[c][e] = 0.f; wv[c][e] = 0.f; bv[c][e] = 0.f; }
        if (ch < nch)
#pragma unroll
            for (int e = 0; e < V; e += 4) { load4f(w + ch * V + e, wv[c] + e); load4f(b + ch * V + e, bv[c] + e); }
    }
    float mu_n = 0.f, rs_n = 0.f;
    if (r0 < nrows) { mu_n = mean[r0]; rs_n = rstd[r0]; }
    int k = 0;
    for (int64_t row = r0; row < nrows; row += G, ++k) {
        const int s = k % DEPTH;
        const float mu = mu_n, rs = rs_n;
        if (row + G < nrows) { mu_n = mean[row + G]; rs_n = rstd[row + G]; }   // next row's stats in flight
        mbar_wait(&rr.bar[s], (k / DEPTH) & 1);
        float xt[CPL][V], g[CPL][V];
        float sg = 0.f, sgx = 0.f;
        uint4 yo[CPL], ho[CPL];
#pragma unroll
        for (int c = 0; c < CPL; ++c) {
            const int ch = lane + 32 * c;
            if (ch < nch) {
                float a[V], u[V], dy[V], gu[V], y[V], dh[V];
                bf16x8_to_f32(*reinterpret_cast<const uint4*>(rr.slot(s, 0) + ch * 16), a);
                bf16x8_to_f32(*reinterpret_cast<const uint4*>(rr.slot(s, 1) + ch * 16), u);
                bf16x8_to_f32(*reinterpret_cast<const uint4*>(rr.slot(s, 2) + ch * 16), dy);
                bf16x8_to_f32(*reinterpret_cast<const uint4*>(rr.slot(s, 3) + ch * 16), gu);
#pragma unroll
                for (int e = 0; e < V; ++e) {
                    xt[c][e] = (a[e] - mu) * rs;
                    const float ah = xt[c][e] * wv[c][e] + bv[c][e];
                    y[e] = ah * u[e];
                    const float dah = dy[e] * u[e];
                    dh[e] = dy[e] * ah * gu[e];
                    g[c][e] = dah * wv[c][e];
                    pw[c][e] += dah * xt[c][e];
                    pb[c][e] += dah;
                    sg += g[c][e];
                    sgx += g[c][e] * xt[c][e];
                }
                Vec<T>::store(reinterpret_cast<T*>(&yo[c]), y);
                Vec<T>::store(reinterpret_cast<T*>(&ho[c]), dh);
            }
        }
        __syncwarp();   // every lane has read slot s
        if (lane == 0 && row + DEPTH * G < nrows) rr.issue(s, src, ldb, row + DEPTH * G);
        const float mg = warp_sum(sg) / d, mgx = warp_sum(sgx) / d;
#pragma unroll
        for (int c = 0; c < CPL; ++c) {
            const int ch = lane + 32 * c;
            if (ch < nch) {
                float o[V];
#pragma unroll
                for (int e = 0; e < V; ++e) o[e] = rs * (g[c][e] - mg - xt[c][e] * mgx);
                Vec<T>::store(dA + row * ldda + ch * V, o);
                *reinterpret_cast<uint4*>(dHU + row * ldh + ch * V) = ho[c];
                if (Y) *reinterpret_cast<uint4*>(Y + row * ldy + ch * V) = yo[c];
            }
        }
    }
    flush_param_grads<T, CPL>(d, pw, pb, dw, db, red);
}

template <int CPL, int DEPTH, bool RES>
__global__ void __launch_bounds__(256) ln_bwd_pipe_k(int64_t nrows, int d, const __nv_bfloat16* __restrict__ dxh,
                                                     int64_t ldg, const __nv_bfloat16* __restrict__ x, int64_t ldx,
                                                     const float* __restrict__ w, const float* __restrict__ mean,
                                                     const float* __restrict__ rstd,
                                                     const __nv_bfloat16* __restrict__ dres, int64_t ldr,
                                                     __nv_bfloat16* __restrict__ dx, int64_t lddx, float* dw, float* db) {
    using T = __nv_bfloat16;
    constexpr int V = 8, NT = RES ? 3 : 2;
    extern __shared__ __align__(128) uint8_t pipe_smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int rb = d * 2, nch = d / V;
    float* red = reinterpret_cast<float*>(pipe_smem);
    uint64_t* bars = reinterpret_cast<uint64_t*>(pipe_smem + 2 * d * 4);
    uint8_t* ring0 = pipe_smem + 2 * d * 4 + kPipeWarps * DEPTH * 8;
    ring0 += (128 - (reinterpret_cast<uintptr_t>(ring0) & 127)) & 127;
    RowRing<NT, DEPTH> rr{ring0 + (size_t)warp * DEPTH * NT * rb, bars + warp * DEPTH, rb};
    const uint8_t* src[3] = {reinterpret_cast<const uint8_t*>(x), reinterpret_cast<const uint8_t*>(dxh),
                             reinterpret_cast<const uint8_t*>(dres)};
    const int64_t ldb[3] = {ldx * 2, ldg * 2, ldr * 2};
    const int64_t G = (int64_t)gridDim.x * kPipeWarps;
    const int64_t r0 = (int64_t)blockIdx.x * kPipeWarps + warp;
    if (lane == 0) {
        for (int s = 0; s < DEPTH; ++s) mbar_init(&rr.bar[s], 1);
        fence_barrier_init();
        for (int s = 0; s < DEPTH; ++s)
            if (r0 + s * G < nrows) rr.issue(s, src, ldb, r0 + s * G);
    }
    __syncwarp();
    float wv[CPL][V], pw[CPL][V], pb[CPL][V];
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
        const int ch = lane + 32 * c;
#pragma unroll
        for (int e = 0; e < V; ++e) { pw[c][e] = 0.f; pb[c][e] = 0.f; wv[c][e] = 0.f; }
        if (ch < nch)
#pragma unroll
            for (int e = 0; e < V; e += 4) load4f(w + ch * V + e, wv[c] + e);
    }
    float mu_n = 0.f, rs_n = 0.f;
    if (r0 < nrows) { mu_n = mean[r0]; rs_n = rstd[r0]; }
    int k = 0;
    for (int64_t row = r0; row < nrows; row += G, ++k) {
        const int s = k % DEPTH;
        const float mu = mu_n, rs = rs_n;
        if (row + G < nrows) { mu_n = mean[row + G]; rs_n = rstd[row + G]; }
        mbar_wait(&rr.bar[s], (k / DEPTH) & 1);
        float xt[CPL][V], g[CPL][V], rv[CPL][V];
        float sg = 0.f, sgx = 0.f;
#pragma unroll
        for (int c = 0; c < CPL; ++c) {
            const int ch = lane + 32 * c;
            if (ch < nch) {
                float xv[V], gv[V];
                bf16x8_to_f32(*reinterpret_cast<const uint4*>(rr.slot(s, 0) + ch * 16), xv);
                bf16x8_to_f32(*reinterpret_cast<const uint4*>(rr.slot(s, 1) + ch * 16), gv);
                if (RES) bf16x8_to_f32(*reinterpret_cast<const uint4*>(rr.slot(s, 2) + ch * 16), rv[c]);
#pragma unroll
                for (int e = 0; e < V; ++e) {
                    xt[c][e] = (xv[e] - mu) * rs;
                    g[c][e] = gv[e] * wv[c][e];
                    pw[c][e] += gv[e] * xt[c][e];
                    pb[c][e] += gv[e];
                    sg += g[c][e];
                    sgx += g[c][e] * xt[c][e];
                }
            }
        }
        __syncwarp();
        if (lane == 0 && row + DEPTH * G < nrows) rr.issue(s, src, ldb, row + DEPTH * G);
        const float mg = warp_sum(sg) / d, mgx = warp_sum(sgx) / d;
#pragma unroll
        for (int c = 0; c < CPL; ++c) {
            const int ch = lane + 32 * c;
            if (ch < nch) {
                float o[V];
#pragma unroll
                for (int e = 0; e < V; ++e) o[e] = rs * (g[c][e] - mg - xt[c][e] * mgx) + (RES ? rv[c][e] : 0.f);
                Vec<T>::store(dx + row * lddx + ch * V, o);
            }
        }
    }
    flush_param_grads<T, CPL>(d, pw, pb, dw, db, red);
}

constexpr int kPipeDepth = 4;
template <int NT>
size_t pipe_smem_bytes(int d) { return (size_t)2 * d * 4 + kPipeWarps * kPipeDepth * 8 + 128 + (size_t)kPipeWarps * kPipeDepth * NT * d * 2; }
// bf16 rows that the bulk copies can stream: 16-byte aligned rows and bases, d <= 512
bool pipe_ok(int d, std::initializer_list<std::pair<const void*, int64_t>> ts) {
    if (d % 8 || d > 512) return false;
    for (auto& t : ts)
        if (t.first && ((reinterpret_cast<uintptr_t>(t.first) & 15) || (t.second % 8))) return false;
    return true;
}

// ------------------------------------------------------------------ column sums / scale
// column sums: a block covers cpb 16-byte column vectors x (256 / cpb) row groups; each thread
// walks its rows with four independent loads in flight, the row groups meet in shared memory,
// and one atomic per column and block reaches global memory
template <typename T>
__global__ void __launch_bounds__(256) colsum_k(int64_t nrows, int n, const T* __restrict__ M, int64_t ldm,
                                                int64_t rows_per_block, int cpb, float* out) {
    constexpr int V = Vec<T>::N;
    __shared__ float red[256 * V];
    const int rgs = 256 / cpb;
    const int cl = threadIdx.x % cpb, rg = threadIdx.x / cpb;
    const int ch = blockIdx.x * cpb + cl;
    const int64_t r0 = blockIdx.y * rows_per_block, r1 = min(nrows, r0 + rows_per_block);
    float s[V] = {};
    if (ch * V < n && rg < rgs) {
        int64_t r = r0 + rg;
        for (; r + 3 * rgs < r1; r += 4 * rgs) {
            float a[V], b[V], c[V], d[V];
            Vec<T>::load(M + r * ldm + ch * V, a);
            Vec<T>::load(M + (r + rgs) * ldm + ch * V, b);
            Vec<T>::load(M + (r + 2 * rgs) * ldm + ch * V, c);
            Vec<T>::load(M + (r + 3 * rgs) * ldm + ch * V, d);
#pragma unroll
            for (int e = 0; e < V; ++e) s[e] += (a[e] + b[e]) + (c[e] + d[e]);
        }
        for (; r < r1; r += rgs) {
            float a[V];
            Vec<T>::load(M + r * ldm + ch * V, a);
#pragma unroll
            for (int e = 0; e < V; ++e) s[e] += a[e];
        }
    }
    if (rgs > 1) {
#pragma unroll
        for (int e = 0; e < V; ++e) red[threadIdx.x * V + e] = s[e];
        __syncthreads();
        if (rg == 0) {
            for (int g = 1; g < rgs; ++g)
#pragma unroll
                for (int e = 0; e < V; ++e) s[e] += red[(g * cpb + cl) * V + e];
        }
    }
    if (rg == 0 && ch * V < n) {
#pragma unroll
        for (int e = 0; e < V; ++e) atomicAdd(out + ch * V + e, s[e]);
    }
}

template <typename T>
int cpl_for(int d) { return (d / Vec<T>::N + 31) / 32; }

int grid_rows(int64_t T) { return (int)((T + kRowsPerBlock - 1) / kRowsPerBlock); }
int grid_persistent(int64_t T) {
    int64_t want = (T + kRowsPerBlock - 1) / kRowsPerBlock;
    int64_t cap = 4LL * num_sms();
    return (int)(want < cap ? (want > 0 ? want : 1) : cap);
}

}  // namespace

// CPL dispatch: chunks-per-lane in {1,2,4,8} covers d up to 1024 (bf16) / 1024 (fp32)
#define UH_CPL_DISPATCH(T, d, ...)                                              \
    do {                                                                        \
        int cpl_ = cpl_for<T>(d);                                               \
        if (cpl_ <= 1) { constexpr int CPL = 1; __VA_ARGS__; }                  \
        else if (cpl_ <= 2) { constexpr int CPL = 2; __VA_ARGS__; }             \
        else if (cpl_ <= 4) { constexpr int CPL = 4; __VA_ARGS__; }             \
        else if (cpl_ <= 8) { constexpr int CPL = 8; __VA_ARGS__; }             \
        else return fail(UH_ERR_UNSUPPORTED, "model dim too large for norm kernels"); \
    } while (0)

// pipelined row kernels: d <= 512 (pipe_ok), one or two 16-byte chunks per lane
#define UH_PIPE_CPL(d, ...)                                                     \
    do {                                                                        \
        if ((d) <= 256) { constexpr int CPL = 1; __VA_ARGS__; }                 \
        else { constexpr int CPL = 2; __VA_ARGS__; }                            \
    } while (0)

#define UH_DT_DISPATCH(dt, ...)                                    \
    do {                                                           \
        if ((dt) == UH_BF16) { using T = __nv_bfloat16; __VA_ARGS__; } \
        else { using T = float; __VA_ARGS__; }                     \
    } while (0)

uh_status ln_fwd(uh_dtype dt, int64_t T_, int d, const void* x, int64_t ldx, const float* w, const float* b, float eps,
                 void* y, int64_t ldy, float* mean, float* rstd, cudaStream_t st) {
    if (T_ == 0) return UH_OK;
    UH_DT_DISPATCH(dt, UH_CPL_DISPATCH(T, d,
        ln_fwd_k<T, CPL><<<grid_rows(T_), 256, 0, st>>>(T_, d, (const T*)x, ldx, w, b, eps, (T*)y, ldy, mean, rstd)));
    note_launch();
    UH_CUDA(cudaGetLastError());
    return UH_OK;
}

uh_status ln_apply(uh_dtype dt, int64_t T_, int d, const void* x, int64_t ldx, const float* w, const float* b,
                   const float* mean, const float* rstd, void* y, int64_t ldy, cudaStream_t st) {
    if (T_ == 0) return UH_OK;
    UH_DT_DISPATCH(dt, UH_CPL_DISPATCH(T, d,
        ln_apply_k<T, CPL><<<grid_rows(T_), 256, 0, st>>>(T_, d, (const T*)x, ldx, w, b, mean, rstd, (T*)y, ldy)));
    note_launch();
    UH_CUDA(cudaGetLastError());
    return UH_OK;
}

uh_status gated_norm_fwd(uh_dtype dt, int64_t T_, int d, const void* A, int64_t lda, const void* U, int64_t ldu,
                         const float* w, const float* b, float eps, void* Y, int64_t ldy, float* mean, float* rstd,
                         cudaStream_t st) {
    if (T_ == 0) return UH_OK;
    UH_DT_DISPATCH(dt, UH_CPL_DISPATCH(T, d,
        gated_fwd_k<T, CPL><<<grid_rows(T_), 256, 0, st>>>(T_, d, (const T*)A, lda, (const T*)U, ldu, w, b, eps,
                                                           (T*)Y, ldy, mean, rstd)));
    note_launch();
    UH_CUDA(cudaGetLastError());
    return UH_OK;
}

uh_status ln_fwd_fp8(int64_t T_, int d, const void* x, int64_t ldx, const float* w, const float* b, float eps,
                     uint8_t* q, int64_t ldq, float* scale, float* mean, float* rstd, cudaStream_t st) {
    if (T_ == 0) return UH_OK;
    UH_CPL_DISPATCH(__nv_bfloat16, d,
        ln_fwd_fp8_k<CPL><<<grid_rows(T_), 256, 0, st>>>(T_, d, (const __nv_bfloat16*)x, ldx, w, b, eps, q, ldq,
                                                         scale, mean, rstd));
    note_launch();
    UH_CUDA(cudaGetLastError());
    return UH_OK;
}

uh_status gated_norm_fwd_fp8(int64_t T_, int d, const void* A, int64_t lda, const void* U, int64_t ldu,
                             const float* w, const float* b, float eps, uint8_t* q, int64_t ldq, float* scale,
                             float* mean, float* rstd, cudaStream_t st) {
    if (T_ == 0) return UH_OK;
    UH_CPL_DISPATCH(__nv_bfloat16, d,
        gated_fwd_fp8_k<CPL><<<grid_rows(T_), 256, 0, st>>>(T_, d, (const __nv_bfloat16*)A, lda,
                                                            (const __nv_bfloat16*)U, ldu, w, b, eps, q, ldq, scale,
                                                            mean, rstd));
    note_launch();
    UH_CUDA(cudaGetLastError());
    return UH_OK;
}

uh_status quant_weight_fp8(int K, int N, const void* W, int64_t ldw, uint8_t* qt, int64_t ldq, float* scale,
                           cudaStream_t st) {
    if (K == 0 || N == 0) return UH_OK;
    quant_weight_fp8_k<<<(N + 31) / 32, 256, 0, st>>>(K, N, (const __nv_bfloat16*)W, ldw, qt, ldq, scale);
    note_launch();
    UH_CUDA(cudaGetLastError());
    return UH_OK;
}

uh_status gated_norm_bwd(uh_dtype dt, int64_t T_, int d, const void* dY, int64_t lddy, const void* A, int64_t lda,
                         const void* U, int64_t ldu, const void* GU, int64_t ldg, const float* w, const float* b,
                         const float* mean, const float* rstd, void* dA, int64_t ldda, void* dHU, int64_t ldh,
                         void* Y, int64_t ldy, float* dw, float* db, cudaStream_t st) {
    if (T_ == 0) return UH_OK;
    if (dt == UH_BF16 && pipe_ok(d, {{dY, lddy}, {A, lda}, {U, ldu}, {GU, ldg}, {dA, ldda}, {dHU, ldh}, {Y, ldy}})) {
        const size_t sm = pipe_smem_bytes<4>(d);
        const int blocks = (int)std::min<int64_t>(2LL * num_sms(), (T_ + kPipeWarps - 1) / kPipeWarps);
        using T = __nv_bfloat16;
        UH_PIPE_CPL(d, {
            UH_CUDA(cudaFuncSetAttribute(gated_bwd_pipe_k<CPL, kPipeDepth>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
            gated_bwd_pipe_k<CPL, kPipeDepth><<<blocks, 256, sm, st>>>(
                T_, d, (const T*)dY, lddy, (const T*)A, lda, (const T*)U, ldu, (const T*)GU, ldg, w, b, mean, rstd,
                (T*)dA, ldda, (T*)dHU, ldh, (T*)Y, ldy, dw, db);
        });
        note_launch();
        UH_CUDA(cudaGetLastError());
        return UH_OK;
    }
    UH_DT_DISPATCH(dt, UH_CPL_DISPATCH(T, d,
        gated_bwd_k<T, CPL><<<grid_persistent(T_), 256, 2 * d * sizeof(float), st>>>(
            T_, d, (const T*)dY, lddy, (const T*)A, lda, (const T*)U, ldu, (const T*)GU, ldg, w, b, mean, rstd,
            (T*)dA, ldda, (T*)dHU, ldh, (T*)Y, ldy, dw, db)));
    note_launch();
    UH_CUDA(cudaGetLastError());
    return UH_OK;
}

uh_status ln_bwd(uh_dtype dt, int64_t T_, int d, const void* dxh, int64_t ldg, const void* x, int64_t ldx,
                 const float* w, const float* mean, const float* rstd, const void* dres, int64_t ldr, void* dx,
                 int64_t lddx, float* dw, float* db, cudaStream_t st) {
    if (T_ == 0) return UH_OK;
    if (dt == UH_BF16 && pipe_ok(d, {{dxh, ldg}, {x, ldx}, {dres, ldr}, {dx, lddx}})) {
        const int blocks = (int)std::min<int64_t>(2LL * num_sms(), (T_ + kPipeWarps - 1) / kPipeWarps);
        using T = __nv_bfloat16;
        if (dres) {
            const size_t sm = pipe_smem_bytes<3>(d);
            UH_PIPE_CPL(d, {
                UH_CUDA(cudaFuncSetAttribute(ln_bwd_pipe_k<CPL, kPipeDepth, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
                ln_bwd_pipe_k<CPL, kPipeDepth, true><<<blocks, 256, sm, st>>>(
                    T_, d, (const T*)dxh, ldg, (const T*)x, ldx, w, mean, rstd, (const T*)dres, ldr, (T*)dx, lddx, dw, db);
            });
        } else {
            const size_t sm = pipe_smem_bytes<2>(d);
            UH_PIPE_CPL(d, {
                UH_CUDA(cudaFuncSetAttribute(ln_bwd_pipe_k<CPL, kPipeDepth, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
                ln_bwd_pipe_k<CPL, kPipeDepth, false><<<blocks, 256, sm, st>>>(
                    T_, d, (const T*)dxh, ldg, (const T*)x, ldx, w, mean, rstd, (const T*)dres, ldr, (T*)dx, lddx, dw, db);
            });
        }
        note_launch();
        UH_CUDA(cudaGetLastError());
        return UH_OK;
    }
    UH_DT_DISPATCH(dt, UH_CPL_DISPATCH(T, d,
        ln_bwd_k<T, CPL><<<grid_persistent(T_), 256, 2 * d * sizeof(float), st>>>(
            T_, d, (const T*)dxh, ldg, (const T*)x, ldx, w, mean, rstd, (const T*)dres, ldr, (T*)dx, lddx, dw, db)));
    note_launch();
    UH_CUDA(cudaGetLastError());
    return UH_OK;
}

uh_status colsum(uh_dtype dt, int64_t T_, int n, const void* M, int64_t ldm, float* out, cudaStream_t st) {
    if (T_ == 0 || n == 0) return UH_OK;
    const int V = dt == UH_BF16 ? 8 : 4;
    const int nch = (n + V - 1) / V;
    int cpb = nch < 256 ? nch : 256;
    while (256 % cpb) ++cpb;                     // row groups tile the block exactly
    const int64_t cols_blocks = (nch + cpb - 1) / cpb;
    int64_t ry = (4 * num_sms() + cols_blocks - 1) / cols_blocks;
    int64_t rpb = (T_ + ry - 1) / ry;
    if (rpb < 64) rpb = 64;
    ry = (T_ + rpb - 1) / rpb;
    dim3 grid((unsigned)cols_blocks, (unsigned)ry);
    UH_DT_DISPATCH(dt, colsum_k<T><<<grid, 256, 0, st>>>(T_, n, (const T*)M, ldm, rpb, cpb, out));
    note_launch();
    UH_CUDA(cudaGetLastError());
    return UH_OK;
}


}  // namespace uh
