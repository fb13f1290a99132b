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

}  // namespace uh
