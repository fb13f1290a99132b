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
// the mask and the rab bias are resolved per 32-column chunk and every
// per-element component is switched on only when some lane of the warp needs it
// (warp-uniform flags, so no divergence):
//   m     per-element mask (the chunk crosses the diagonal, the band edge, or L)
//   pp    per-element position bias (the chunk is within P-1 of the diagonal)
//   tmode 0: the time bucket is constant along every lane's chunk
//         1: at most two buckets per lane -> one threshold compare per element
//         2: generic per-element bucket (only right next to the diagonal)
// Buckets of floor(log2 dt) are monotone along a row because timestamps are
// sorted, so a lane's chunk has buckets b_first..b_last and "two buckets" means
// one threshold on the column timestamp.  rab tables live in smem (pos_s: P
// floats, ts_s: NB <= 32 floats).  Rows beyond L are "don't care" (their outputs
// are never stored) and never force a per-element component.
// Column timestamps are carried per lane as 32-bit offsets from the chunk's
// first column (chunks must span < 2^31 s).
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

UH_DEV int32_t clamp_i32(int64_t v) {
    return (int32_t)(v < -1 ? -1 : (v > 0x7fffffffLL ? 0x7fffffffLL : v));
}

// tcol: this lane's column timestamp t[col0 + lane] (prefetched one tile ahead by the caller)
UH_DEV int64_t col_time(const ChunkCtx& c, int col0, int lane) {
    return c.ts_s ? __ldg(c.t + imin(col0 + lane, c.L - 1)) : 0;
}

struct Chunk {
    bool m, pp;       // warp-uniform: per-element mask / position bias needed
    int tmode;        // warp-uniform: 0 constant bucket, 1 threshold, 2 generic
    float bias;       // per lane: constant part of the bias (pos[P-1] and ts[b_base])
    float tdelta;     // per lane (tmode 1): ts[b_other] - ts[b_base]
    int32_t thr;      // per lane (tmode 1): column offset threshold of the b_other side
    int32_t rel;      // per lane: this lane's column timestamp - chunk base
    int b_base, b_other;
    int64_t tcol;     // per lane: column timestamp (tmode 2)
};

// rows are queries (forward, dQ); columns are keys kb..kb+31 (dt decreasing along the row)
UH_DEV Chunk q_chunk(const ChunkCtx& c, int qp, bool qok, int64_t tq, int kb, int lane, int64_t tcol) {
    Chunk r;
    const bool full = (kb + 31 <= qp) && (qp - kb <= c.K1 || kb + 31 < c.K2);
    bool pp = false;
    float bias = 0.f;
    if (c.pos_s) {
        pp = qp - kb - 31 < c.P - 1;
        bias += c.pos_s[c.P - 1];
    }
    int tm = 0;
    r.tdelta = 0.f; r.thr = -1; r.rel = 0; r.b_base = 0; r.b_other = 0; r.tcol = tcol;
    if (c.ts_s) {
        const int64_t base = shfl64(tcol, 0);
        const int bf = time_bucket(tq - base, c.NB);                 // first column: largest dt
        const int bl = time_bucket(tq - shfl64(tcol, 31), c.NB);     // last column: smallest dt
        r.b_base = bl; r.b_other = bf;
        r.rel = clamp_i32(tcol - base);
        tm = bf == bl ? 0 : (bf == bl + 1 ? 1 : 2);
        if (tm == 1) {
            r.tdelta = c.ts_s[bf] - c.ts_s[bl];
            r.thr = clamp_i32(tq - (int64_t(1) << bf) - base);     // column in b_other iff rel <= thr
        }
        bias += c.ts_s[bl];
    }
    r.m = __any_sync(0xffffffffu, qok && !full);
    r.pp = __any_sync(0xffffffffu, qok && pp);
    const int t1 = __any_sync(0xffffffffu, qok && tm >= 1), t2 = __any_sync(0xffffffffu, qok && tm == 2);
    r.tmode = t2 ? 2 : (t1 ? 1 : 0);
    r.bias = bias;
    return r;
}

// rows are keys (dK/dV); columns are queries qb..qb+31 (dt increasing along the row)
UH_DEV Chunk k_chunk(const ChunkCtx& c, int kp, bool kok, int64_t tk, int qb, int lane, int64_t tcol) {
    Chunk r;
    const bool full = (qb >= kp) && (qb + 31 < c.L) && (qb + 31 - kp <= c.K1 || kp < c.K2);
    bool pp = false;
    float bias = 0.f;
    if (c.pos_s) {
        pp = qb - kp < c.P - 1;
        bias += c.pos_s[c.P - 1];
    }
    int tm = 0;
    r.tdelta = 0.f; r.thr = 0x7fffffff; r.rel = 0; r.b_base = 0; r.b_other = 0; r.tcol = tcol;
    if (c.ts_s) {
        const int64_t base = shfl64(tcol, 0);
        const int bf = time_bucket(base - tk, c.NB);                 // first column: smallest dt
        const int bl = time_bucket(shfl64(tcol, 31) - tk, c.NB);     // last column: largest dt
        r.b_base = bf; r.b_other = bl;
        r.rel = clamp_i32(tcol - base);
        tm = bf == bl ? 0 : (bl == bf + 1 ? 1 : 2);
        if (tm == 1) {
            r.tdelta = c.ts_s[bl] - c.ts_s[bf];
            r.thr = clamp_i32(tk + (int64_t(1) << bl) - base);     // column in b_other iff rel >= thr
        }
        bias += c.ts_s[bf];
    }
    r.m = __any_sync(0xffffffffu, kok && !full);
    r.pp = __any_sync(0xffffffffu, kok && pp);
    const int t1 = __any_sync(0xffffffffu, kok && tm >= 1), t2 = __any_sync(0xffffffffu, kok && tm == 2);
    r.tmode = t2 ? 2 : (t1 ? 1 : 0);
    r.bias = bias;
    return r;
}

// x[c] = alpha * s[c] + rab(c) for a query-row chunk; returns the per-element bucket
// in bk[] only when tmode == 2 (else bk is untouched).  Masking is separate (q_mask).
template <bool WANT_BUCKET>
UH_DEV void q_bias(const ChunkCtx& c, const Chunk& ch, int qp, int64_t tq, int kb, const float* s, float* x,
                   bool* other, int* bk) {
#pragma unroll
    for (int j = 0; j < 32; ++j) x[j] = fmaf(s[j], c.alpha, ch.bias);
    if (ch.pp) {
        const float pl = c.pos_s[c.P - 1];
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            int dd = qp - kb - j;
            dd = dd < 0 ? 0 : (dd < c.P - 1 ? dd : c.P - 1);
            x[j] += c.pos_s[dd] - pl;
        }
    }
    if (ch.tmode == 1) {
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            const bool o = __shfl_sync(0xffffffffu, ch.rel, j) <= ch.thr;
            if (WANT_BUCKET) other[j] = o;
            x[j] += o ? ch.tdelta : 0.f;
        }
    } else if (ch.tmode == 2) {
        const float tb = c.ts_s[ch.b_base];
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            const int b = time_bucket(tq - shfl64(ch.tcol, j), c.NB);
            if (WANT_BUCKET) bk[j] = b;
            x[j] += c.ts_s[b] - tb;
        }
    }
}

// the same for a key-row chunk (columns are queries)
UH_DEV void k_bias(const ChunkCtx& c, const Chunk& ch, int kp, int64_t tk, int qb, const float* s, float* x) {
#pragma unroll
    for (int j = 0; j < 32; ++j) x[j] = fmaf(s[j], c.alpha, ch.bias);
    if (ch.pp) {
        const float pl = c.pos_s[c.P - 1];
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            int dd = qb + j - kp;
            dd = dd < 0 ? 0 : (dd < c.P - 1 ? dd : c.P - 1);
            x[j] += c.pos_s[dd] - pl;
        }
    }
    if (ch.tmode == 1) {
#pragma unroll
        for (int j = 0; j < 32; ++j) x[j] += (__shfl_sync(0xffffffffu, ch.rel, j) >= ch.thr) ? ch.tdelta : 0.f;
    } else if (ch.tmode == 2) {
        const float tb = c.ts_s[ch.b_base];
#pragma unroll
        for (int j = 0; j < 32; ++j) x[j] += c.ts_s[time_bucket(shfl64(ch.tcol, j) - tk, c.NB)] - tb;
    }
}

// per-element visibility (only called when ch.m)
UH_DEV bool q_visible(const ChunkCtx& c, int qp, bool qok, int kp) {
    return qok && kp < c.L && mask_ok(qp, kp, c.K1, c.K2);
}
UH_DEV bool k_visible(const ChunkCtx& c, int kp, bool kok, int qp) {
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
