# attention (bf16 path): 32-bit timestamps relative to each sequence's first, built once per call
# into the workspace (rel_ts_k), so the epilogues' column / row timestamp loads are 4-byte loads
# with no 64-bit subtract and clamp
COMMON = [
    ("attn_common.cuh", "    const int64_t* t;\n", "    const int64_t* t;\n    const int32_t* t32;   // bf16 path: timestamps relative to the sequence start (rel_ts_k)\n"),
    ("attn_common.cuh", "    const int64_t* t;    // timestamps of this sequence (t + seq_start)",
     "    const int32_t* t;    // relative 32-bit timestamps of this sequence (t32 + seq_start)"),
    ("attn_common.cuh", "    return c.ts_h ? rel32(__ldg(c.t + imin(col0 + lane, c.L - 1)), c.t0) : 0;",
     "    return c.ts_h ? __ldg(c.t + imin(col0 + lane, c.L - 1)) : 0;"),
    ("attn_common.cuh", "    c.t = a.t ? a.t + o : nullptr;\n    c.t0 = a.ts ? __ldg(a.t + o) : 0;",
     "    c.t = a.t32 ? a.t32 + o : nullptr;\n    c.t0 = 0;"),
]
FWD = [
    ("attn_fwd_sm100.cu", """        int64_t t0n = 0, tqn = 0;    // the next item's first timestamp and this row's (raw)
        auto load_rowtimes = [&](const WorkItem& x) {
            if (a.ts) {
                t0n = __ldg(a.t + x.seq_start);
                tqn = __ldg(a.t + x.seq_start + imin(x.tile * BM + r, x.seq_len - 1));
            }
        };""", """        int32_t tqn = 0;    // the next item's timestamp of this row (relative)
        auto load_rowtimes = [&](const WorkItem& x) {
            if (a.ts) tqn = __ldg(a.t32 + x.seq_start + imin(x.tile * BM + r, x.seq_len - 1));
        };"""),
    ("attn_fwd_sm100.cu", """            cx.t = a.t ? a.t + o : nullptr;
            cx.t0 = a.ts ? t0n : 0;""", """            cx.t = a.t32 ? a.t32 + o : nullptr;
            cx.t0 = 0;"""),
    ("attn_fwd_sm100.cu", "const int32_t tq = (a.ts && qok) ? rel32(tqn, cx.t0) : 0;", "const int32_t tq = (a.ts && qok) ? tqn : 0;"),
    ("attn_fwd_sm100.cu", "                    const int64_t* tp = a.t + on;", "                    const int32_t* tp = a.t32 + on;"),
]
BWD = [
    ("attn_bwd_sm100.cu", "const int32_t tk = (a.ts && kok) ? rel32(__ldg(a.t + o + kp), cx.t0) : 0;",
     "const int32_t tk = (a.ts && kok) ? __ldg(a.t32 + o + kp) : 0;"),
]
ATTN = [
    ("attn.cu", "    size_t items_q = 0, counters = 0, pos_ext = 0, dq_acc = 0, total = 0;",
     "    size_t items_q = 0, counters = 0, pos_ext = 0, t32 = 0, dq_acc = 0, total = 0;"),
    ("attn.cu", """    if (backward && dt == UH_BF16) {   // fp32 dQ accumulator [T, H dh]""",
     """    if (dt == UH_BF16 && desc->time_bias) {   // relative 32-bit timestamps [T]
        w.t32 = off;
        off += align256((size_t)jag->total_tokens * sizeof(int32_t));
    }
    if (backward && dt == UH_BF16) {   // fp32 dQ accumulator [T, H dh]"""),
    ("attn.cu", """static uh_status build_pos_ext(const AttnCall& c, const WsLayout& w, AttnArgs& a) {""",
     """// t32[i] = clamp(t[i] - t[start of i's sequence], 0, 2^31 - 1): one block per sequence
__global__ void __launch_bounds__(256) rel_ts_k(const int32_t* __restrict__ off, const int64_t* __restrict__ t,
                                                int32_t* __restrict__ t32) {
    const int b = blockIdx.x;
    const int o0 = off[b], o1 = off[b + 1];
    if (o1 <= o0) return;
    const int64_t t0 = t[o0];
    for (int i = o0 + threadIdx.x; i < o1; i += blockDim.x) {
        const int64_t d = t[i] - t0;
        t32[i] = (int32_t)(d < 0 ? 0 : (d > 0x7fffffffLL ? 0x7fffffffLL : d));
    }
}

static uh_status build_t32(const AttnCall& c, const WsLayout& w, AttnArgs& a) {
    if (!a.ts || !a.t || c.jag->num_seqs == 0) return UH_OK;
    int32_t* t32 = reinterpret_cast<int32_t*>((uint8_t*)c.ws + w.t32);
    a.t32 = t32;
    rel_ts_k<<<c.jag->num_seqs, 256, 0, c.st>>>(c.jag->offsets, a.t, t32);
    note_launch();
    UH_CUDA(cudaGetLastError());
    return UH_OK;
}

static uh_status build_pos_ext(const AttnCall& c, const WsLayout& w, AttnArgs& a) {"""),
    ("attn.cu", """    if (dt == UH_F32) return attn_fwd_simt_launch(a, c.st);
    UH_TRY(build_pos_ext(c, w, a));""", """    if (dt == UH_F32) return attn_fwd_simt_launch(a, c.st);
    UH_TRY(build_pos_ext(c, w, a));
    UH_TRY(build_t32(c, w, a));"""),
    ("attn.cu", """    UH_TRY(schedule(c, dt, SCHED_K, (WorkItem*)a.items, a.counter));
    UH_TRY(build_pos_ext(c, w, a));""", """    UH_TRY(schedule(c, dt, SCHED_K, (WorkItem*)a.items, a.counter));
    UH_TRY(build_pos_ext(c, w, a));
    UH_TRY(build_t32(c, w, a));"""),
]
PATCHES = COMMON + FWD + BWD + ATTN
