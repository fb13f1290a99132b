// attn.cu — F0 (the jagged tile schedule) and the attention dispatch.
//
// F0 runs on the device: one block counts the work items of every sequence
// (P:190 fully jagged, no padding), buckets them by cost (number of visited
// 128-wide tiles under the SLA mask) and writes them cost-descending
// (LPT order for the persistent kernels).  No host->device copy is involved, so
// every call is stream-ordered and CUDA-graph capturable.
#include <cub/block/block_scan.cuh>

#include "attn_common.cuh"
#include "internal.h"

namespace uh {

uh_status attn_fwd_simt_launch(const AttnArgs& a, cudaStream_t st);
uh_status attn_bwd_simt_launch(const AttnArgs& a, cudaStream_t st);
uh_status attn_fwd_sm100_launch(const AttnArgs& a, cudaStream_t st, int64_t T);
uh_status attn_bwd_sm100_launch(const AttnArgs& akv, cudaStream_t st, int64_t T);

namespace {

enum { SCHED_Q = 0, SCHED_K = 1 };
constexpr int kSchedThreads = 1024;
constexpr int kCostBuckets = 4096;

__host__ __device__ inline int item_cost(int mode, int t, int L, int BMt, int BNt, int K1, int K2) {
    if (mode == SCHED_Q) return key_tiles_count(key_tiles(t * BMt, BMt, L, K1, K2, BNt));
    const int k0 = t * BMt;
    return (query_end(k0, BMt, L, K1, K2) - k0 + BNt - 1) / BNt;
}

// one block: the query-tile (forward) or key-tile (backward) schedule of the batch
__global__ void __launch_bounds__(kSchedThreads) build_schedule_k(const int32_t* __restrict__ offsets, int B, int H,
                                                                  int BMt, int BNt, int K1, int K2, int mode,
                                                                  WorkItem* __restrict__ items, int* counter) {
    using Scan = cub::BlockScan<int, kSchedThreads>;
    __shared__ int hist[kCostBuckets];
    __shared__ typename Scan::TempStorage tmp;
    constexpr int PER = kCostBuckets / kSchedThreads;
    for (int i = threadIdx.x; i < kCostBuckets; i += kSchedThreads) hist[i] = 0;
    if (threadIdx.x == 0 && counter) *counter = 0;
    __syncthreads();
    // one warp per sequence, lanes over its tiles (long sequences have hundreds of tiles);
    // under SLA nearly every tile has the same cost: aggregate equal buckets per warp first
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int b = warp; b < B; b += kSchedThreads / 32) {
        const int L = offsets[b + 1] - offsets[b];
        const int nt = (L + BMt - 1) / BMt;
        for (int t0 = 0; t0 < nt; t0 += 32) {
            const int t = t0 + lane;
            const bool on = t < nt;
            int c = on ? item_cost(mode, t, L, BMt, BNt, K1, K2) : -1;
            c = c < kCostBuckets - 1 ? c : kCostBuckets - 1;
            const unsigned peers = __match_any_sync(0xffffffffu, c);
            if (on && lane == __ffs(peers) - 1) atomicAdd(&hist[c], __popc(peers));
        }
    }
    __syncthreads();
    // exclusive scan in DESCENDING cost order: bucket c starts after all buckets c' > c
    int v[PER], sum = 0;
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        v[i] = hist[kCostBuckets - 1 - (threadIdx.x * PER + i)];
        sum += v[i];
    }
    int excl;
    Scan(tmp).ExclusiveSum(sum, excl);
    __syncthreads();
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        hist[kCostBuckets - 1 - (threadIdx.x * PER + i)] = excl * H;
        excl += v[i];
    }
    __syncthreads();
    for (int b = warp; b < B; b += kSchedThreads / 32) {
        const int o = offsets[b], L = offsets[b + 1] - o;
        const int nt = (L + BMt - 1) / BMt;
        for (int t0 = 0; t0 < nt; t0 += 32) {
            const int t = t0 + lane;
            const bool on = t < nt;
            int c = on ? item_cost(mode, t, L, BMt, BNt, K1, K2) : -1;
            c = c < kCostBuckets - 1 ? c : kCostBuckets - 1;
            const unsigned peers = __match_any_sync(0xffffffffu, c);
            const int leader = __ffs(peers) - 1;
            int base = 0;
            if (on && lane == leader) base = atomicAdd(&hist[c], __popc(peers) * H);
            base = __shfl_sync(0xffffffffu, base, leader);
            if (on) {
                const int pos = base + __popc(peers & ((1u << lane) - 1)) * H;
                for (int h = 0; h < H; ++h) items[pos + h] = WorkItem{o, L, t, h};
            }
        }
    }
}

int64_t count_items(const uh_jagged* jag, int BMt, int H) {
    int64_t n = 0;
    for (int b = 0; b < jag->num_seqs; ++b) {
        int64_t L = jag->host_offsets[b + 1] - jag->host_offsets[b];
        n += (L + BMt - 1) / BMt;
    }
    return n * H;
}

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

struct WsLayout {
    size_t items_q = 0, counters = 0, pos_ext = 0, dq_acc = 0, total = 0;
    int pos_ext_len = 0;
};

int tile_rows(uh_dtype dt) { return dt == UH_BF16 ? 128 : 64; }

WsLayout ws_layout(const uh_jagged* jag, const uh_attn_desc* desc, uh_dtype dt, int backward) {
    WsLayout w;
    const int BMt = tile_rows(dt);
    const int64_t n = count_items(jag, BMt, desc->num_heads);
    size_t off = 0;
    w.items_q = off; off += align256(n * sizeof(WorkItem));
    w.counters = off; off += 256;
    if (dt == UH_BF16 && desc->pos_bias) {   // two copies of the extended position table (attn_common.cuh)
        w.pos_ext_len = (jag->max_len + 2 * kPosOff + 3) & ~3;   // copy 1 stays 16-byte aligned
        w.pos_ext = off;
        off += align256((size_t)2 * w.pos_ext_len * sizeof(float));
    }
    if (backward && dt == UH_BF16) {   // fp32 dQ accumulator [T, H dh]
        w.dq_acc = off;
        off += align256((size_t)jag->total_tokens * desc->num_heads * desc->head_dim * sizeof(float));
    }
    w.total = off;
    return w;
}

}  // namespace

size_t attn_ws_bytes(const uh_jagged* jag, uh_mask m, const uh_attn_desc* desc, uh_dtype dt, int backward) {
    (void)m;
    return ws_layout(jag, desc, dt, backward).total;
}

// Extended position table for the tcgen05 epilogues (R7; layout in attn_common.cuh): copy c, index i
// holds (pos[clamp(i + c - kPosOff, 0, P - 1)] - pos[P - 1]) / 2.
__global__ void __launch_bounds__(256) rab_ext_k(const float* __restrict__ pos, int P, float* __restrict__ ext, int Lt) {
    const float far = pos[P - 1];
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < 2 * Lt; i += gridDim.x * blockDim.x) {
        const int c = i >= Lt ? 1 : 0;
        int dd = i - c * Lt + c - kPosOff;
        dd = dd < 0 ? 0 : (dd > P - 1 ? P - 1 : dd);
        ext[i] = 0.5f * (pos[dd] - far);
    }
}

static uh_status build_pos_ext(const AttnCall& c, const WsLayout& w, AttnArgs& a) {
    if (!w.pos_ext_len) return UH_OK;
    a.pos_ext = reinterpret_cast<float*>((uint8_t*)c.ws + w.pos_ext);
    a.pos_ext_len = w.pos_ext_len;
    const int n = 2 * w.pos_ext_len;
    rab_ext_k<<<(n + 255) / 256 < 64 ? (n + 255) / 256 : 64, 256, 0, c.st>>>(a.pos, a.P, const_cast<float*>(a.pos_ext),
                                                                            w.pos_ext_len);
    note_launch();
    UH_CUDA(cudaGetLastError());
    return UH_OK;
}

static AttnArgs base_args(const AttnCall& c, uh_dtype dt) {
    AttnArgs a{};
    a.H = c.desc->num_heads;
    a.dh = c.desc->head_dim;
    a.alpha = c.desc->alpha;
    a.inv_n = 1.0f / c.desc->norm_n;
    a.K1 = c.mask.window;
    a.K2 = c.mask.n_global;
    a.pos = c.desc->pos_bias; a.P = c.desc->pos_bias_len;
    a.ts = c.desc->time_bias; a.NB = c.desc->time_bias_len;
    a.t = c.desc->timestamps;
    a.q = c.q; a.k = c.k; a.v = c.v; a.ld_qkv = c.ld_qkv;
    a.out = c.out; a.ld_out = c.ld_out;
    a.dout = c.dout; a.ld_dout = c.ld_dout;
    a.dq = c.dq; a.dk = c.dk; a.dv = c.dv; a.ld_grad = c.ld_grad;
    a.gq = c.gq; a.gk = c.gk; a.gv = c.gv; a.ld_gate = c.ld_gate;
    a.dpos = c.dpos; a.dts = c.dts;
    a.T = c.jag->total_tokens;
    (void)dt;
    return a;
}

static uh_status schedule(const AttnCall& c, uh_dtype dt, int mode, WorkItem* items, int* counter) {
    const int BMt = tile_rows(dt);
    const int BNt = dt == UH_BF16 ? 128 : 32;
    build_schedule_k<<<1, kSchedThreads, 0, c.st>>>(c.jag->offsets, c.jag->num_seqs, c.desc->num_heads,
                                                                 BMt, BNt, c.mask.window, c.mask.n_global, mode,
                                                                 items, counter);
    note_launch();
    UH_CUDA(cudaGetLastError());
    return UH_OK;
}

uh_status attn_fwd_run(const AttnCall& c, uh_dtype dt) {
    const WsLayout w = ws_layout(c.jag, c.desc, dt, 0);
    uint8_t* ws = (uint8_t*)c.ws;
    AttnArgs a = base_args(c, dt);
    a.items = (const WorkItem*)(ws + w.items_q);
    a.counter = (int*)(ws + w.counters);
    a.n_items = (int)count_items(c.jag, tile_rows(dt), a.H);
    if (a.n_items == 0) return UH_OK;
    UH_TRY(schedule(c, dt, SCHED_Q, (WorkItem*)a.items, a.counter));
    if (dt == UH_F32) return attn_fwd_simt_launch(a, c.st);
    UH_TRY(build_pos_ext(c, w, a));
    return attn_fwd_sm100_launch(a, c.st, c.jag->total_tokens);
}

uh_status attn_bwd_run(const AttnCall& c, uh_dtype dt) {
    const WsLayout w = ws_layout(c.jag, c.desc, dt, 1);
    uint8_t* ws = (uint8_t*)c.ws;
    AttnArgs a = base_args(c, dt);
    a.items = (const WorkItem*)(ws + w.items_q);
    a.counter = (int*)(ws + w.counters);
    a.n_items = (int)count_items(c.jag, tile_rows(dt), a.H);
    if (a.n_items == 0) return UH_OK;
    if (dt == UH_F32) {
        UH_TRY(schedule(c, dt, SCHED_Q, (WorkItem*)a.items, nullptr));
        return attn_bwd_simt_launch(a, c.st);
    }
    // bf16: the key-tile schedule (one key-major fused kernel) and the fp32 dQ accumulator
    a.dq_acc = reinterpret_cast<float*>(ws + w.dq_acc);
    a.ld_acc = (int64_t)a.H * a.dh;
    UH_TRY(schedule(c, dt, SCHED_K, (WorkItem*)a.items, a.counter));
    UH_TRY(build_pos_ext(c, w, a));
    return attn_bwd_sm100_launch(a, c.st, c.jag->total_tokens);
}

}  // namespace uh
