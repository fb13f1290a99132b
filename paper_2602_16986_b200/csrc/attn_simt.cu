// attn_simt.cu — fp32 SIMT "verification build" of the jagged SLA HSTU attention
// (Eq. 3; SLA P:140-146), forward and backward.  FFMA with accurate expf:
// TF32 tensor cores cannot meet the 1e-4 bar of the north star.
//
// Forward / dQ kernels: one block per (sequence, head, 64-query tile); 4 threads per
// query row, each owning dh/4 of the head dims; key tiles of 32 rows staged in smem.
// dK/dV kernel: one block per (sequence, head, 64-key tile), queries staged in smem.
#include <climits>

#include "attn_common.cuh"
#include "internal.h"

namespace uh {
namespace {

constexpr int SQ = 64;  // rows per block
constexpr int SK = 32;  // staged rows per tile

__device__ __forceinline__ float red4(float v) {
    v += __shfl_xor_sync(0xffffffffu, v, 1);
    v += __shfl_xor_sync(0xffffffffu, v, 2);
    return v;
}

template <int DH>
__global__ void __launch_bounds__(256) attn_fwd_simt(AttnArgs a) {
    constexpr int DPT = DH / 4;
    __shared__ float Ks[SK][DH], Vs[SK][DH];
    __shared__ int64_t ts_k[SK];
    const WorkItem it = a.items[blockIdx.x];
    const int L = it.seq_len, o = it.seq_start, h = it.head & 0xFFFF;
    const int q0 = it.tile * SQ;
    const int r = threadIdx.x >> 2, part = threadIdx.x & 3;
    const int qp = q0 + r;
    const bool qok = qp < L;
    const float* Q = (const float*)a.q;
    const float* K = (const float*)a.k;
    const float* V = (const float*)a.v;
    float qv[DPT], acc[DPT];
#pragma unroll
    for (int j = 0; j < DPT; ++j) {
        qv[j] = qok ? Q[(int64_t)(o + qp) * a.ld_qkv + h * DH + part * DPT + j] : 0.f;
        acc[j] = 0.f;
    }
    const int64_t tq = (a.ts && qok) ? a.t[o + qp] : 0;
    KeyTiles kt = key_tiles(q0, SQ, L, a.K1, a.K2, SK);
    const int nt = key_tiles_count(kt);
    for (int i = 0; i < nt; ++i) {
        const int k0 = key_tile_at(kt, i) * SK;
        __syncthreads();
        for (int e = threadIdx.x; e < SK * DH; e += 256) {
            int kk = e / DH, c = e % DH;
            bool ok = k0 + kk < L;
            int64_t row = (int64_t)(o + k0 + kk);
            Ks[kk][c] = ok ? K[row * a.ld_qkv + h * DH + c] : 0.f;
            Vs[kk][c] = ok ? V[row * a.ld_qkv + h * DH + c] : 0.f;
        }
        if (a.ts && threadIdx.x < SK) ts_k[threadIdx.x] = (k0 + threadIdx.x < L) ? a.t[o + k0 + threadIdx.x] : 0;
        __syncthreads();
        for (int kk = 0; kk < SK; ++kk) {
            float dot = 0.f;
#pragma unroll
            for (int j = 0; j < DPT; ++j) dot = fmaf(qv[j], Ks[kk][part * DPT + j], dot);
            dot = red4(dot);
            const int kp = k0 + kk;
            if (!qok || kp >= L || !mask_ok(qp, kp, a.K1, a.K2)) continue;
            float s = a.alpha * dot + rab_bias(a, qp, kp, tq, a.ts ? ts_k[kk] : 0);
            float p = s / (1.0f + expf(-s)) * a.inv_n;
#pragma unroll
            for (int j = 0; j < DPT; ++j) acc[j] = fmaf(p, Vs[kk][part * DPT + j], acc[j]);
        }
    }
    if (qok) {
        float* out = (float*)a.out;
#pragma unroll
        for (int j = 0; j < DPT; ++j) out[(int64_t)(o + qp) * a.ld_out + h * DH + part * DPT + j] = acc[j];
    }
}

// dQ (and drab): per query row, loop over visible keys.
template <int DH>
__global__ void __launch_bounds__(256) attn_dq_simt(AttnArgs a) {
    constexpr int DPT = DH / 4;
    __shared__ float Ks[SK][DH], Vs[SK][DH];
    __shared__ int64_t ts_k[SK];
    __shared__ float dts_s[64];
    const WorkItem it = a.items[blockIdx.x];
    const int L = it.seq_len, o = it.seq_start, h = it.head & 0xFFFF;
    const int q0 = it.tile * SQ;
    const int r = threadIdx.x >> 2, part = threadIdx.x & 3;
    const int qp = q0 + r;
    const bool qok = qp < L;
    const float* Q = (const float*)a.q;
    const float* K = (const float*)a.k;
    const float* V = (const float*)a.v;
    const float* dA = (const float*)a.dout;
    if (threadIdx.x < 64) dts_s[threadIdx.x] = 0.f;
    float qv[DPT], gv[DPT], acc[DPT];
#pragma unroll
    for (int j = 0; j < DPT; ++j) {
        const int c = h * DH + part * DPT + j;
        qv[j] = qok ? Q[(int64_t)(o + qp) * a.ld_qkv + c] : 0.f;
        gv[j] = qok ? dA[(int64_t)(o + qp) * a.ld_dout + c] : 0.f;
        acc[j] = 0.f;
    }
    const int64_t tq = (a.ts && qok) ? a.t[o + qp] : 0;
    KeyTiles kt = key_tiles(q0, SQ, L, a.K1, a.K2, SK);
    const int nt = key_tiles_count(kt);
    for (int i = 0; i < nt; ++i) {
        const int k0 = key_tile_at(kt, i) * SK;
        __syncthreads();
        for (int e = threadIdx.x; e < SK * DH; e += 256) {
            int kk = e / DH, c = e % DH;
            bool ok = k0 + kk < L;
            int64_t row = (int64_t)(o + k0 + kk);
            Ks[kk][c] = ok ? K[row * a.ld_qkv + h * DH + c] : 0.f;
            Vs[kk][c] = ok ? V[row * a.ld_qkv + h * DH + c] : 0.f;
        }
        if (a.ts && threadIdx.x < SK) ts_k[threadIdx.x] = (k0 + threadIdx.x < L) ? a.t[o + k0 + threadIdx.x] : 0;
        __syncthreads();
        for (int kk = 0; kk < SK; ++kk) {
            float dot = 0.f, dp = 0.f;
#pragma unroll
            for (int j = 0; j < DPT; ++j) {
                dot = fmaf(qv[j], Ks[kk][part * DPT + j], dot);
                dp = fmaf(gv[j], Vs[kk][part * DPT + j], dp);
            }
            dot = red4(dot);
            dp = red4(dp);
            const int kp = k0 + kk;
            if (!qok || kp >= L || !mask_ok(qp, kp, a.K1, a.K2)) continue;
            const int64_t tk = a.ts ? ts_k[kk] : 0;
            float s = a.alpha * dot + rab_bias(a, qp, kp, tq, tk);
            float sg = 1.0f / (1.0f + expf(-s));
            float ds = dp * sg * (1.0f + s * (1.0f - sg)) * a.inv_n;
#pragma unroll
            for (int j = 0; j < DPT; ++j) acc[j] = fmaf(a.alpha * ds, Ks[kk][part * DPT + j], acc[j]);
            if (part == 0) {
                if (a.dpos) { int dd = qp - kp; atomicAdd(a.dpos + (dd < a.P - 1 ? dd : a.P - 1), ds); }
                if (a.dts) atomicAdd(&dts_s[time_bucket(tq - tk, a.NB)], ds);
            }
        }
    }
    if (qok) {
        float* dq = (float*)a.dq;
        const float* g = (const float*)a.gq;
#pragma unroll
        for (int j = 0; j < DPT; ++j) {
            const int c = h * DH + part * DPT + j;
            float v = acc[j];
            if (g) v *= g[(int64_t)(o + qp) * a.ld_gate + c];
            dq[(int64_t)(o + qp) * a.ld_grad + c] = v;
        }
    }
    __syncthreads();
    if (a.dts && threadIdx.x < a.NB && threadIdx.x < 64) atomicAdd(a.dts + threadIdx.x, dts_s[threadIdx.x]);
}

// dK, dV: per key row, loop over the queries that see it.
template <int DH>
__global__ void __launch_bounds__(256) attn_dkv_simt(AttnArgs a) {
    constexpr int DPT = DH / 4;
    __shared__ float Qs[SK][DH], Gs[SK][DH];
    __shared__ int64_t ts_q[SK];
    const WorkItem it = a.items[blockIdx.x];
    const int L = it.seq_len, o = it.seq_start, h = it.head & 0xFFFF;
    const int k0 = it.tile * SQ;
    const int r = threadIdx.x >> 2, part = threadIdx.x & 3;
    const int kp = k0 + r;
    const bool kok = kp < L;
    const float* Q = (const float*)a.q;
    const float* K = (const float*)a.k;
    const float* V = (const float*)a.v;
    const float* dA = (const float*)a.dout;
    float kv[DPT], vv[DPT], dk[DPT], dv[DPT];
#pragma unroll
    for (int j = 0; j < DPT; ++j) {
        const int c = h * DH + part * DPT + j;
        kv[j] = kok ? K[(int64_t)(o + kp) * a.ld_qkv + c] : 0.f;
        vv[j] = kok ? V[(int64_t)(o + kp) * a.ld_qkv + c] : 0.f;
        dk[j] = 0.f; dv[j] = 0.f;
    }
    const int64_t tk = (a.ts && kok) ? a.t[o + kp] : 0;
    const int qend = query_end(k0, SQ, L, a.K1, a.K2);
    for (int qt = k0; qt < qend; qt += SK) {
        __syncthreads();
        for (int e = threadIdx.x; e < SK * DH; e += 256) {
            int qq = e / DH, c = e % DH;
            bool ok = qt + qq < L;
            int64_t row = (int64_t)(o + qt + qq);
            Qs[qq][c] = ok ? Q[row * a.ld_qkv + h * DH + c] : 0.f;
            Gs[qq][c] = ok ? dA[row * a.ld_dout + h * DH + c] : 0.f;
        }
        if (a.ts && threadIdx.x < SK) ts_q[threadIdx.x] = (qt + threadIdx.x < L) ? a.t[o + qt + threadIdx.x] : 0;
        __syncthreads();
        for (int qq = 0; qq < SK; ++qq) {
            float dot = 0.f, dp = 0.f;
#pragma unroll
            for (int j = 0; j < DPT; ++j) {
                dot = fmaf(kv[j], Qs[qq][part * DPT + j], dot);
                dp = fmaf(vv[j], Gs[qq][part * DPT + j], dp);
            }
            dot = red4(dot);
            dp = red4(dp);
            const int qp = qt + qq;
            if (!kok || qp >= L || !mask_ok(qp, kp, a.K1, a.K2)) continue;
            float s = a.alpha * dot + rab_bias(a, qp, kp, a.ts ? ts_q[qq] : 0, tk);
            float sg = 1.0f / (1.0f + expf(-s));
            float p = s * sg * a.inv_n;
            float ds = dp * sg * (1.0f + s * (1.0f - sg)) * a.inv_n;
#pragma unroll
            for (int j = 0; j < DPT; ++j) {
                dv[j] = fmaf(p, Gs[qq][part * DPT + j], dv[j]);
                dk[j] = fmaf(a.alpha * ds, Qs[qq][part * DPT + j], dk[j]);
            }
        }
    }
    if (kok) {
        float* DK = (float*)a.dk;
        float* DV = (float*)a.dv;
        const float* gk = (const float*)a.gk;
        const float* gv = (const float*)a.gv;
#pragma unroll
        for (int j = 0; j < DPT; ++j) {
            const int c = h * DH + part * DPT + j;
            const int64_t rr = (int64_t)(o + kp);
            float x = dk[j], y = dv[j];
            if (gk) x *= gk[rr * a.ld_gate + c];
            if (gv) y *= gv[rr * a.ld_gate + c];
            DK[rr * a.ld_grad + c] = x;
            DV[rr * a.ld_grad + c] = y;
        }
    }
}

}  // namespace

// items: one per (sequence, head, 64-row tile)
uh_status attn_fwd_simt_launch(const AttnArgs& a, cudaStream_t st) {
    if (a.n_items == 0) return UH_OK;
    switch (a.dh) {
        case 32: attn_fwd_simt<32><<<a.n_items, 256, 0, st>>>(a); break;
        case 64: attn_fwd_simt<64><<<a.n_items, 256, 0, st>>>(a); break;
        case 128: attn_fwd_simt<128><<<a.n_items, 256, 0, st>>>(a); break;
        default: return fail(UH_ERR_SHAPE, "fp32 attention: head_dim must be 32, 64 or 128");
    }
    note_launch();
    UH_CUDA(cudaGetLastError());
    return UH_OK;
}

uh_status attn_bwd_simt_launch(const AttnArgs& a, cudaStream_t st) {
    if (a.n_items == 0) return UH_OK;
    switch (a.dh) {
        case 32: attn_dq_simt<32><<<a.n_items, 256, 0, st>>>(a); attn_dkv_simt<32><<<a.n_items, 256, 0, st>>>(a); break;
        case 64: attn_dq_simt<64><<<a.n_items, 256, 0, st>>>(a); attn_dkv_simt<64><<<a.n_items, 256, 0, st>>>(a); break;
        case 128: attn_dq_simt<128><<<a.n_items, 256, 0, st>>>(a); attn_dkv_simt<128><<<a.n_items, 256, 0, st>>>(a); break;
        default: return fail(UH_ERR_SHAPE, "fp32 attention: head_dim must be 32, 64 or 128");
    }
    note_launch();
    note_launch();
    UH_CUDA(cudaGetLastError());
    return UH_OK;
}

}  // namespace uh
