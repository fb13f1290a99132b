// attn_common.cuh — mask / bias / tile-range helpers shared by the CUDA attention
// kernels (fp32 SIMT twin and tcgen05 kernels).  Mask: SLA in the
// time-ascending reading R1-R4 of DESIGN.md:  k <= q  and  (q-k <= K1  or  k < K2).
#pragma once
#include <stdint.h>

#include "sm100.cuh"

namespace uh {

#define UH_HD __host__ __device__ __forceinline__
UH_HD int imin(int a, int b) { return a < b ? a : b; }
UH_HD int imax(int a, int b) { return a > b ? a : b; }

// Work item of the jagged tile schedule (F0): one (sequence, head, row tile).
struct WorkItem {
    int32_t seq_start;  // first token row of the sequence
    int32_t seq_len;    // L
    int32_t tile;       // row tile index within the sequence (query tile fwd, key tile bwd)
    int32_t head;       // head index (high 16 bits: split index for the bwd global tiles)
};

struct AttnArgs {
    const WorkItem* items;
    int n_items;
    int H, dh;
    float alpha, inv_n;
    int K1, K2;  // K1 = INT32_MAX => full causal
    const float* pos; int P;
    const float* ts; int NB;
    const int64_t* t;
    const void *q, *k, *v; int64_t ld_qkv;
    void* out; int64_t ld_out;            // forward output A
    const void* dout; int64_t ld_dout;    // backward: dA
    void *dq, *dk, *dv; int64_t ld_grad;  // backward outputs
    const void *gq, *gk, *gv; int64_t ld_gate;  // optional gates (silu'(h)) multiplied into dq/dk/dv
    float* dq_acc; int64_t ld_acc;        // fp32 dQ accumulator (tcgen05 bwd)
    float *dpos, *dts;
    int* counter;                          // dynamic work counter (persistent kernels)
};

UH_HD bool mask_ok(int q, int k, int K1, int K2) {
    return k <= q && (q - k <= K1 || k < K2);
}

UH_DEV int time_bucket(int64_t dt, int NB) {
    if (dt < 1) dt = 1;
    int b = 63 - __clzll((unsigned long long)dt);
    return b < NB - 1 ? b : NB - 1;
}

// additive relative position/time bias rab(q,k) (R7); q,k positions in the sequence
UH_DEV float rab_bias(const AttnArgs& a, int q, int k, int64_t tq, int64_t tk) {
    float r = 0.f;
    if (a.pos) { int dd = q - k; dd = dd < 0 ? 0 : (dd < a.P - 1 ? dd : a.P - 1); r += __ldg(a.pos + dd); }
    if (a.ts) r += __ldg(a.ts + time_bucket(tq - tk, a.NB));
    return r;
}

// Key tiles (width BN) visible from query rows [q0, q0+rows) of a length-L sequence:
// global tiles [0, g_end) followed by band tiles [b_begin, b_end), de-duplicated.
struct KeyTiles { int g_end, b_begin, b_end; };
UH_HD KeyTiles key_tiles(int q0, int rows, int L, int K1, int K2, int BN) {
    KeyTiles r;
    int qlast = imin(q0 + rows, L) - 1;
    int lo = (K1 >= qlast) ? 0 : imax(0, q0 - K1);
    r.b_begin = lo / BN;
    r.b_end = qlast / BN + 1;
    int gk = imin(K2, qlast + 1);
    r.g_end = imin((gk + BN - 1) / BN, r.b_begin);
    return r;
}
UH_HD int key_tiles_count(const KeyTiles& r) { return r.g_end + (r.b_end - r.b_begin); }
UH_HD int key_tile_at(const KeyTiles& r, int i) { return i < r.g_end ? i : r.b_begin + (i - r.g_end); }

// Query rows that can see key rows [k0, k0+rows): [k0, qend)
UH_HD int query_end(int k0, int rows, int L, int K1, int K2) {
    int klast = imin(k0 + rows, L) - 1;
    if (k0 < K2) return L;  // a global key is visible to every later query
    long long e = (long long)klast + K1 + 1;
    return e < L ? (int)e : L;
}

// ----------------------------------------------------------------------------
// 32-column chunks of a score tile, seen by one thread-row (tcgen05 epilogues).
//
// The epilogue budget is ~8 lane-ops per score element at full tensor rate, so
// the mask and the rab bias are resolved per 32-column chunk: when every lane of
// the warp has a fully visible chunk with a constant position bucket and a
// constant time bucket (the common case away from the diagonal and the band
// edge), the whole chunk takes the fast path "x = alpha*S + bias_lane".  Otherwise
// the warp evaluates mask and bias per element.  rab tables live in smem
// (pos_s: P floats, ts_s: NB floats).  Rows beyond L are "don't care" (their
// outputs are never stored) and never force the slow path.
// ----------------------------------------------------------------------------
struct ChunkCtx {
    const float* pos_s; int P;
    const float* ts_s; int NB;
    const int64_t* t;   // timestamps of this sequence (t + seq_start) or nullptr
    int K1, K2, L;
    float alpha;
};

UH_DEV int64_t shfl64(int64_t v, int src) {
    int lo = __shfl_sync(0xffffffffu, (int)(v & 0xffffffff), src);
    int hi = __shfl_sync(0xffffffffu, (int)(v >> 32), src);
    return ((int64_t)hi << 32) | (uint32_t)lo;
}

// rows are queries (forward, dQ); columns are keys kb..kb+31
struct QChunk {
    bool uni;        // warp-uniform fast path
    float bias;      // per-lane constant bias on the fast path
    int b0;          // time bucket of the chunk's first column (constant on the fast path)
    int64_t tcol;    // this lane's column timestamp (for the slow path)
};
// tcol: this lane's column timestamp t[col0 + lane] (prefetched one tile ahead by the caller)
UH_DEV int64_t col_time(const ChunkCtx& c, int col0, int lane) {
    return c.ts_s ? __ldg(c.t + imin(col0 + lane, c.L - 1)) : 0;
}
UH_DEV QChunk q_chunk(const ChunkCtx& c, int qp, bool qok, int64_t tq, int kb, int lane, int64_t tcol) {
    QChunk r;
    bool full = (kb + 31 <= qp) && (qp - kb <= c.K1 || kb + 31 < c.K2);
    bool uni = full;
    float bias = 0.f;
    if (c.pos_s) {
        uni = uni && (qp - kb - 31 >= c.P - 1);
        bias += c.pos_s[c.P - 1];
    }
    r.tcol = 0;
    r.b0 = 0;
    if (c.ts_s) {
        r.tcol = tcol;
        const int b0 = time_bucket(tq - shfl64(r.tcol, 0), c.NB);
        const int b1 = time_bucket(tq - shfl64(r.tcol, 31), c.NB);
        uni = uni && b0 == b1;
        bias += c.ts_s[b0];
        r.b0 = b0;
    }
    r.uni = __all_sync(0xffffffffu, uni || !qok);
    r.bias = bias;
    return r;
}
// slow path for one element of a query-row chunk: returns false when masked
UH_DEV bool q_elem(const ChunkCtx& c, const QChunk& ch, int qp, bool qok, int64_t tq, int kb, int j, float& bias,
                   int& bkt) {
    const int kp = kb + j;
    const int64_t tk = c.ts_s ? shfl64(ch.tcol, j) : 0;
    bias = 0.f;
    bkt = 0;
    if (c.pos_s) { int dd = qp - kp; dd = dd < 0 ? 0 : (dd < c.P - 1 ? dd : c.P - 1); bias += c.pos_s[dd]; }
    if (c.ts_s) { bkt = time_bucket(tq - tk, c.NB); bias += c.ts_s[bkt]; }
    return qok && kp < c.L && mask_ok(qp, kp, c.K1, c.K2);
}
UH_DEV bool q_elem(const ChunkCtx& c, const QChunk& ch, int qp, bool qok, int64_t tq, int kb, int j, float& bias) {
    int b;
    return q_elem(c, ch, qp, qok, tq, kb, j, bias, b);
}

// rows are keys (dK/dV); columns are queries qb..qb+31
UH_DEV QChunk k_chunk(const ChunkCtx& c, int kp, bool kok, int64_t tk, int qb, int lane, int64_t tcol) {
    QChunk r;
    bool full = (qb >= kp) && (qb + 31 < c.L) && (qb + 31 - kp <= c.K1 || kp < c.K2);
    bool uni = full;
    float bias = 0.f;
    if (c.pos_s) {
        uni = uni && (qb - kp >= c.P - 1);
        bias += c.pos_s[c.P - 1];
    }
    r.tcol = 0;
    r.b0 = 0;
    if (c.ts_s) {
        r.tcol = tcol;
        const int b0 = time_bucket(shfl64(r.tcol, 0) - tk, c.NB);
        const int b1 = time_bucket(shfl64(r.tcol, 31) - tk, c.NB);
        uni = uni && b0 == b1;
        bias += c.ts_s[b0];
        r.b0 = b0;
    }
    r.uni = __all_sync(0xffffffffu, uni || !kok);
    r.bias = bias;
    return r;
}
UH_DEV bool k_elem(const ChunkCtx& c, const QChunk& ch, int kp, bool kok, int64_t tk, int qb, int j, float& bias) {
    const int qp = qb + j;
    const int64_t tq = c.ts_s ? shfl64(ch.tcol, j) : 0;
    bias = 0.f;
    if (c.pos_s) { int dd = qp - kp; dd = dd < 0 ? 0 : (dd < c.P - 1 ? dd : c.P - 1); bias += c.pos_s[dd]; }
    if (c.ts_s) bias += c.ts_s[time_bucket(tq - tk, c.NB)];
    return kok && qp < c.L && mask_ok(qp, kp, c.K1, c.K2);
}

// Stage the rab tables into shared memory (all threads of the CTA; caller syncs).
UH_DEV void stage_rab(const AttnArgs& a, float* pos_s, float* ts_s) {
    if (a.pos)
        for (int i = threadIdx.x; i < a.P; i += blockDim.x) pos_s[i] = __ldg(a.pos + i);
    if (a.ts)
        for (int i = threadIdx.x; i < a.NB; i += blockDim.x) ts_s[i] = __ldg(a.ts + i);
}

constexpr int kMaxPosSmem = 2048;  // bf16 tcgen05 path: pos_bias_len <= 2048 (validated)

}  // namespace uh
