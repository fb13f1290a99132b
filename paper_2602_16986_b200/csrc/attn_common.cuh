// attn_common.cuh — mask / bias / tile-range helpers shared by the CUDA attention
// kernels (fp32 SIMT twin and tcgen05 kernels).  Mask: SLA in the
// time-ascending reading R1-R4 of DESIGN.md:  k <= q  and  (q-k <= K1  or  k < K2).
#pragma once
#include <stdint.h>

#include "sm100.cuh"

namespace uh {

#if UH_TRACE
// timestamps of CTA 0 for timeline analysis (trace builds only: -DUH_TRACE=1)
__device__ long long* g_trace = nullptr;
// the pointer is read once per kernel into a register: a global load per trace point
// would add an L2 round trip to every traced interval
#define TRACE_SETUP() long long* const uh_tr_ = blockIdx.x == 0 ? g_trace : nullptr
#define TRACE(slot) do { if (uh_tr_ && (slot) < 8192) uh_tr_[(slot)] = clock64(); } while (0)
#else
#define TRACE_SETUP() do { } while (0)
#define TRACE(slot) do { } while (0)
#endif

// Checked builds (-DUH_CHECKED=1, tools/build_variant.py checked): device-side range checks on
// the work items, table indices, reduction targets and output rows; a violation traps the
// kernel (compute-sanitizer is not available on the GPU pool, so these are the bounds checks)
#if UH_CHECKED
#define UH_CHECK(cond) do { if (!(cond)) __trap(); } while (0)
#else
#define UH_CHECK(cond) do { } while (0)
#endif

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
    int64_t T;                             // total tokens (checked builds)
    int H, dh;
    float alpha, inv_n;
    int K1, K2;  // K1 = INT32_MAX => full causal
    const float* pos; int P;
    const float* pos_ext; int pos_ext_len;  // bf16 path: two copies of the extended position table (rab_ext_*)
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

// checked builds: a work item lies inside its sequence and the batch
UH_DEV void check_item(const AttnArgs& a, const WorkItem& it, int rows) {
    UH_CHECK(it.seq_start >= 0 && it.seq_len > 0 && (int64_t)it.seq_start + it.seq_len <= a.T);
    UH_CHECK(it.tile >= 0 && it.tile * rows < it.seq_len && (it.head & 0xFFFF) < a.H);
}

// MMA block order of one item with n tiles whose second block (PV / dQ / dV-dK) runs LAG
// tiles behind its first (S, or S and dP): S0 .. S(LAG-1), then S(j) P(j-LAG) pairs, then
// the remaining P blocks.  Lets the issuer name (and probe) the barrier of block k+1.
struct MmaBlk { int tile; bool first; };
UH_HD MmaBlk lag_block(int k, int n, int lag) {
    const int h = n < lag ? n : lag;
    if (k < h) return {k, true};
    int r = k - h;
    const int pairs = n > lag ? n - lag : 0;
    if (r < 2 * pairs) return {(r & 1) ? (r >> 1) : lag + (r >> 1), !(r & 1)};
    return {pairs + (r - 2 * pairs), false};
}

// Dynamic work distribution for the persistent tcgen05 kernels: the producer lane claims
// the next item of the cost-descending list (F0) with one atomicAdd, so the list is served
// longest-first to whichever CTA frees up (LPT), and publishes it to the CTA's other roles
// through a small shared-memory ring (mbarrier full/empty per slot).  -1 ends the stream.
constexpr int kItemRing = 4;
struct ItemRing {
    uint64_t full[kItemRing], empty[kItemRing];
    int idx[kItemRing];
};
UH_DEV void ring_init(ItemRing* r, int consumer_warps);
UH_DEV int ring_claim_publish(ItemRing* r, int k, int* counter, int n_items);
UH_DEV int ring_take(ItemRing* r, int k, int lane);

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
// The epilogue budget is a few lane-ops per score element at full tensor rate, so
// the mask and the rab bias are resolved per 32-column chunk and every
// per-element component is switched on only when some lane of the warp needs it
// (warp-uniform flags from one redux.or, so no divergence):
//   FLAG_M   per-element mask (the chunk crosses the diagonal, the band edge, or L)
//   FLAG_P   per-element position bias (some element is within P-1 of the diagonal):
//            pairs of consecutive offsets read as one 8-byte load from the extended
//            table in global memory (L1-resident), any P (R7)
//   FLAG_T1  some lane sees two time buckets: the columns of the larger-dt bucket
//            form a prefix (queries as rows) / suffix (keys as rows) whose length a
//            5-step binary search over the lanes' column timestamps finds
//   FLAG_T2  some lane sees >2 buckets (right next to the diagonal): per element
// Buckets floor(log2 dt) are monotone along a row because timestamps are sorted.
// Everything carries h = x/2 (x = alpha S + rab), the argument of tanh in
// silu(x) = h + h tanh(h); tables are pre-halved.  Timestamps are 32-bit offsets
// from the sequence's first timestamp (a sequence must span < 2^31 s).
// Rows beyond L are "don't care" in the forward (never stored) and never raise a flag there; in the
// backward a key row beyond L raises FLAG_M, whose visibility mask zeroes its h and dP (dS = 0).
//
// Extended position table (built per call by rab_ext_k, attn.cu): two copies of
// length Lt = max_len + 2 kPosOff, copy c holding e_c[i] = (pos[clamp(i + c - kPosOff,
// 0, P-1)] - pos[P-1]) / 2, so offset dd maps to index dd + kPosOff; a lane whose pairs
// start at an odd index reads copy 1, making every pair load 8-byte aligned.
// ----------------------------------------------------------------------------
constexpr int kPosOff = 128;       // extended table covers dd in [-kPosOff, max_len + kPosOff)
enum { FLAG_M = 1, FLAG_P = 2, FLAG_T1 = 4, FLAG_T2 = 8 };

struct ChunkCtx {
    const float* pe;     // global: extended table copy 0 at offset kPosOff (pe[dd] for dd >= -kPosOff), or nullptr
    int Lt;              // length of one copy (copy 1 = pe + Lt)
    float pos_far;       // pos[P-1] / 2
    int P;
    const float* ts_h;   // smem: ts / 2, or nullptr
    int NB;
    const int64_t* t;    // timestamps of this sequence (t + seq_start)
    int64_t t0;          // first timestamp of the sequence (32-bit offsets are relative to it)
    int K1, K2, L;
    float ha;            // alpha / 2
};

UH_DEV int32_t rel32(int64_t t, int64_t t0) {
    int64_t d = t - t0;
    return (int32_t)(d < 0 ? 0 : (d > 0x7fffffffLL ? 0x7fffffffLL : d));
}
UH_DEV int bucket32(int32_t dt, int NB) {  // min(NB-1, floor(log2(max(dt,1))))
    const int b = 31 - __clz(dt < 1 ? 1 : dt);
    return b < NB - 1 ? b : NB - 1;
}
// column timestamp of this lane for the chunk starting at col0 (prefetched a tile ahead)
UH_DEV int32_t col_time(const ChunkCtx& c, int col0, int lane) {
    return c.ts_h ? rel32(__ldg(c.t + imin(col0 + lane, c.L - 1)), c.t0) : 0;
}

struct Chunk {
    unsigned flags;   // warp-uniform OR of FLAG_*
    float hbias;      // per lane: constant part of h's bias (pos_far + ts_h[b_base])
    float hbias_o;    // per lane: bias of the "other" time bucket (FLAG_T1)
    int n;            // per lane (FLAG_T1): q-rows: columns [0,n) are in the other bucket;
                      //                      k-rows: columns [n,32) are in the other bucket
    int b_base, b_other;
    int bd;           // per lane: clamped qp-kb (q-rows) / qb-kp (k-rows) for the position table
    int32_t tcol;     // per lane: column timestamp (32-bit offset)
};

// number of lanes c whose value v[c] (non-decreasing in c) satisfies v[c] <= x (less=false) or v[c] < x (less=true)
template <bool LESS>
UH_DEV int count_le(int32_t v, int32_t x) {
    int lo = 0;
#pragma unroll
    for (int step = 16; step >= 1; step >>= 1) {
        const int32_t w = __shfl_sync(0xffffffffu, v, lo + step - 1);
        if (LESS ? (w < x) : (w <= x)) lo += step;
    }
    // lo in [0, 31]; include lane 31 if it also satisfies
    const int32_t w = __shfl_sync(0xffffffffu, v, 31);
    if (lo == 31 && (LESS ? (w < x) : (w <= x))) lo = 32;
    return lo;
}

// rows are queries (forward); columns are keys kb..kb+31 (dt decreasing along the row)
UH_DEV Chunk q_chunk(const ChunkCtx& c, int qp, bool qok, int32_t tq, int kb, int32_t tcol) {
    Chunk r;
    unsigned f = 0;
    if (!((kb + 31 <= qp) && (qp - kb <= c.K1 || kb + 31 < c.K2))) f |= FLAG_M;
    float hb = 0.f;
    r.bd = 0;
    if (c.pe) {
        const int d0 = qp - kb;                      // offsets d0 - j, j = 0..31
        if (d0 - 31 < c.P - 1) f |= FLAG_P;
        r.bd = d0 < -64 ? -64 : (d0 > c.L + 64 ? c.L + 64 : d0);
        hb += c.pos_far;
    }
    r.tcol = tcol;
    r.b_base = r.b_other = 0;
    r.hbias_o = 0.f;
    r.n = 0;
    int32_t thr = 0;
    if (c.ts_h) {
        const int bf = bucket32(tq - __shfl_sync(0xffffffffu, tcol, 0), c.NB);   // first column: largest dt
        const int bl = bucket32(tq - __shfl_sync(0xffffffffu, tcol, 31), c.NB);  // last column: smallest dt
        r.b_base = bl; r.b_other = bf;
        if (bf == bl + 1) f |= FLAG_T1;
        else if (bf > bl + 1) f |= FLAG_T2;
        const int64_t th = (int64_t)tq - ((int64_t)1 << bf);                   // other bucket iff tcol <= th
        thr = (int32_t)(th < -1 ? -1 : th);
        r.hbias_o = hb + c.ts_h[bf];
        hb += c.ts_h[bl];
    }
    r.flags = __reduce_or_sync(0xffffffffu, qok ? f : 0u);
    if (r.flags & FLAG_T1) {
        const int cnt = count_le<false>(tcol, thr);   // all lanes take part in the shuffles
        r.n = (r.b_other == r.b_base + 1) ? cnt : 0;
    }
    r.hbias = hb;
    return r;
}

// rows are keys (backward); columns are queries qb..qb+31 (dt increasing along the row)
UH_DEV Chunk k_chunk(const ChunkCtx& c, int kp, bool kok, int32_t tk, int qb, int32_t tcol) {
    Chunk r;
    unsigned f = 0;
    if (!((qb >= kp) && (qb + 31 < c.L) && (qb + 31 - kp <= c.K1 || kp < c.K2))) f |= FLAG_M;
    float hb = 0.f;
    r.bd = 0;
    if (c.pe) {
        const int d0 = qb - kp;                      // offsets d0 + j, j = 0..31
        if (d0 < c.P - 1) f |= FLAG_P;
        r.bd = d0 < -96 ? -96 : (d0 > c.L + 64 ? c.L + 64 : d0);
        hb += c.pos_far;
    }
    r.tcol = tcol;
    r.b_base = r.b_other = 0;
    r.hbias_o = 0.f;
    r.n = 32;
    int32_t thr = 0;
    if (c.ts_h) {
        const int bf = bucket32(__shfl_sync(0xffffffffu, tcol, 0) - tk, c.NB);   // first column: smallest dt
        const int bl = bucket32(__shfl_sync(0xffffffffu, tcol, 31) - tk, c.NB);  // last column: largest dt
        r.b_base = bf; r.b_other = bl;
        if (bl == bf + 1) f |= FLAG_T1;
        else if (bl > bf + 1) f |= FLAG_T2;
        const int64_t th = (int64_t)tk + ((int64_t)1 << bl);                   // other bucket iff tcol >= th
        thr = (int32_t)(th > 0x7fffffffLL ? 0x7fffffffLL : th);
        r.hbias_o = hb + c.ts_h[bl];
        hb += c.ts_h[bf];
    }
    r.flags = __reduce_or_sync(0xffffffffu, kok ? f : (unsigned)FLAG_M);   // keys beyond L: masked
    if (r.flags & FLAG_T1) {
        const int cnt = count_le<true>(tcol, thr);    // all lanes take part in the shuffles
        r.n = (r.b_other == r.b_base + 1) ? cnt : 32;
    }
    r.hbias = hb;
    return r;
}

// 8-byte load of two consecutive extended-table entries (L1-cached, read-only)
UH_DEV float2 pe_pair(const float* p) { return __ldg(reinterpret_cast<const float2*>(p)); }

// h[j] = (alpha S + rab)/2 for a 32-column chunk as one FFMA2 per pair of columns, the pair's
// bias built in registers: the chunk's constant (pos_far + ts of the base bucket), the other
// bucket's constant on the columns past the FLAG_T1 split, the position-table pair (FLAG_P), and
// per-element buckets for FLAG_T2.  Q_ROWS: rows are queries, columns keys kb + j (offsets bd - j,
// the other bucket on columns [0, n)); else rows are keys, columns queries qb + j (offsets bd + j,
// the other bucket on columns [n, 32)).
template <bool Q_ROWS, bool T1, bool P>
UH_DEV void chunk_h_pairs(const ChunkCtx& c, const Chunk& ch, const float* s, float* h) {
    const uint64_t A2 = f2_pack(c.ha, c.ha);
    const float hb = ch.hbias, ho = ch.hbias_o;
    const float* pe = nullptr;
    if (P) {   // q rows: pairs (j, j+1) = offsets (bd-j, bd-j-1), one aligned pair at bd-j-1; k rows: at bd+j
        const int i0 = Q_ROWS ? ch.bd - 1 + kPosOff : ch.bd + kPosOff;
        UH_CHECK(Q_ROWS ? (i0 - 31 >= 0 && i0 + 1 < c.Lt) : (i0 >= 0 && i0 + 33 < c.Lt));
        pe = c.pe - kPosOff + (i0 & 1) * c.Lt + (i0 & ~1);   // copy (i0 & 1), even index
    }
#pragma unroll
    for (int j = 0; j < 32; j += 2) {
        float b0 = hb, b1 = hb;
        if (T1) {
            b0 = (Q_ROWS ? j < ch.n : j >= ch.n) ? ho : hb;
            b1 = (Q_ROWS ? j + 1 < ch.n : j + 1 >= ch.n) ? ho : hb;
        }
        uint64_t B2 = f2_pack(b0, b1);
        if (P) {
            const float2 pp = pe_pair(Q_ROWS ? pe - j : pe + j);
            B2 = fadd2(B2, Q_ROWS ? f2_pack(pp.y, pp.x) : f2_pack(pp.x, pp.y));
        }
        const float2 v = f2_unpack(ffma2(f2_pack(s[j], s[j + 1]), A2, B2));
        h[j] = v.x; h[j + 1] = v.y;
    }
}

template <bool Q_ROWS>
UH_DEV void chunk_h(const ChunkCtx& c, const Chunk& ch, int32_t trow, const float* s, float* h) {
    const bool t1 = ch.flags & FLAG_T1, p = ch.flags & FLAG_P;   // warp-uniform
    if (t1) {
        if (p) chunk_h_pairs<Q_ROWS, true, true>(c, ch, s, h); else chunk_h_pairs<Q_ROWS, true, false>(c, ch, s, h);
    } else {
        if (p) chunk_h_pairs<Q_ROWS, false, true>(c, ch, s, h); else chunk_h_pairs<Q_ROWS, false, false>(c, ch, s, h);
    }
    if (ch.flags & FLAG_T2) {   // > 2 buckets in some row: per element, relative to the base bucket's bias
        const float tb = c.ts_h[ch.b_base];
        const bool multi = !(ch.b_other == ch.b_base + 1 || ch.b_other == ch.b_base);
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            const int32_t tc = __shfl_sync(0xffffffffu, ch.tcol, j);
            const int b = bucket32(Q_ROWS ? trow - tc : tc - trow, c.NB);
            h[j] += multi ? c.ts_h[b] - tb : 0.f;
        }
    }
}

// query-row chunk (forward)
UH_DEV void q_h(const ChunkCtx& c, const Chunk& ch, int32_t tq, const float* s, float* h) {
    chunk_h<true>(c, ch, tq, s, h);
}
// key-row chunk (backward)
UH_DEV void k_h(const ChunkCtx& c, const Chunk& ch, int32_t tk, const float* s, float* h) {
    chunk_h<false>(c, ch, tk, s, h);
}

// Visibility of a 32-column chunk as a bit mask (bit c = column c visible), for FLAG_M
// chunks: causal, window and global-prefix bounds are column ranges, so the mask costs a
// few integer ops per chunk instead of a predicate per element.
UH_DEV uint32_t bit_range(int lo, int hi) {   // bits [lo, hi] of 0..31 (empty if hi < lo)
    lo = lo < 0 ? 0 : lo;
    hi = hi > 31 ? 31 : hi;
    if (hi < lo) return 0u;
    const uint32_t up = hi == 31 ? 0xFFFFFFFFu : ((2u << hi) - 1u);
    return up & ~((1u << lo) - 1u);
}
constexpr int kHugeWindow = 0x40000000;   // K1 at or beyond this is "full causal"
// query row qp, key columns kb..kb+31 (k <= q < L, so the length bound is implied)
UH_DEV uint32_t q_vis_bits(const ChunkCtx& c, int qp, bool qok, int kb) {
    if (!qok) return 0u;
    const int d = qp - kb;                                            // column of k == q
    const uint32_t win = c.K1 >= kHugeWindow ? 0xFFFFFFFFu : bit_range(d - c.K1, 31);
    return bit_range(0, d) & (win | bit_range(0, c.K2 - kb - 1));
}
// key row kp, query columns qb..qb+31
UH_DEV uint32_t k_vis_bits(const ChunkCtx& c, int kp, bool kok, int qb) {
    if (!kok) return 0u;
    const int d = kp - qb;                                            // column of q == k
    const uint32_t win = (kp < c.K2 || c.K1 >= kHugeWindow) ? 0xFFFFFFFFu : bit_range(0, d + c.K1);
    return bit_range(d, 31) & win & bit_range(0, c.L - qb - 1);
}
// zero the fp32 values of invisible columns (before they are packed to bf16)
UH_DEV void apply_vis(float* v, uint32_t m) {
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = (m >> j) & 1u ? v[j] : 0.f;
}

// per-element visibility (only needed when FLAG_M)
UH_DEV bool q_visible(const ChunkCtx& c, int qp, bool qok, int kp) {
    return qok && kp < c.L && mask_ok(qp, kp, c.K1, c.K2);
}
UH_DEV bool k_visible(const ChunkCtx& c, int kp, bool kok, int qp) {
    return kok && qp < c.L && mask_ok(qp, kp, c.K1, c.K2);
}

// row r of a [rows x 64] bf16 K-major SW128 tile: 32 packed columns (16 x bf16x2) at col0 (0 or 32)
UH_DEV void store_row32_packed(uint8_t* tile, int r, int col0, const uint32_t* v) {
    uint8_t* row = tile + r * 128;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        const int ch = (col0 >> 3) + c;
        *reinterpret_cast<uint4*>(row + ((ch ^ (r & 7)) << 4)) =
            make_uint4(v[4 * c + 0], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
    }
}
// zero element j (low half for even j, high half for odd j) of a packed bf16x2 array
UH_DEV void zero_half(uint32_t* v, int j) { v[j >> 1] &= (j & 1) ? 0x0000FFFFu : 0xFFFF0000u; }
// sum of 16 packed bf16x2 values, pairwise in bf16x2, final pair in fp32
UH_DEV float sum_packed16(const uint32_t* v) {
    uint32_t a[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = add_bf16x2(v[i], v[i + 8]);
#pragma unroll
    for (int i = 0; i < 4; ++i) a[i] = add_bf16x2(a[i], a[i + 4]);
    a[0] = add_bf16x2(a[0], a[2]); a[1] = add_bf16x2(a[1], a[3]);
    const float2 x = unpack_bf16x2(a[0]), y = unpack_bf16x2(a[1]);
    return (x.x + x.y) + (y.x + y.y);
}

// Stage the pre-halved time-bias table into shared memory (all threads; caller syncs).
UH_DEV void stage_ts(const AttnArgs& a, float* ts_h) {
    if (a.ts)
        for (int i = threadIdx.x; i < a.NB; i += blockDim.x) ts_h[i] = 0.5f * __ldg(a.ts + i);
}

UH_DEV ChunkCtx make_ctx(const AttnArgs& a, const float* ts_h, int o, int L) {
    ChunkCtx c;
    c.pe = a.pos ? a.pos_ext + kPosOff : nullptr;
    c.Lt = a.pos_ext_len;
    c.pos_far = a.pos ? 0.5f * __ldg(a.pos + a.P - 1) : 0.f;
    c.P = a.P;
    c.ts_h = a.ts ? ts_h : nullptr;
    c.NB = a.NB;
    c.t = a.t ? a.t + o : nullptr;
    c.t0 = a.ts ? __ldg(a.t + o) : 0;
    c.K1 = a.K1; c.K2 = a.K2; c.L = L;
    c.ha = 0.5f * a.alpha;
    return c;
}


UH_DEV void ring_init(ItemRing* r, int consumer_warps) {
    for (int i = 0; i < kItemRing; ++i) { mbar_init(&r->full[i], 1); mbar_init(&r->empty[i], consumer_warps); }
}
// producer lane: claim, publish (the slot is free once every consumer warp has read it)
UH_DEV int ring_claim_publish(ItemRing* r, int k, int* counter, int n_items) {
    const int s = k % kItemRing;
    mbar_wait_sleep(&r->empty[s], ((k / kItemRing) & 1) ^ 1);
    const int w = atomicAdd(counter, 1);
    r->idx[s] = w < n_items ? w : -1;
    mbar_arrive(&r->full[s]);   // release: the index is visible to the waiting roles
    return w < n_items ? w : -1;
}
// whole warp: the k-th item of this CTA (or -1)
UH_DEV int ring_take(ItemRing* r, int k, int lane) {
    const int s = k % kItemRing;
    mbar_wait_sleep(&r->full[s], (k / kItemRing) & 1);
    const int w = *reinterpret_cast<volatile int*>(&r->idx[s]);
    __syncwarp();
    if (lane == 0) mbar_arrive(&r->empty[s]);
    return w;
}

}  // namespace uh
