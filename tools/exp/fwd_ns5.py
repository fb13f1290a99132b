# fwd (4 warpgroups): five S buffers (S0..S4 | O at 320 | Q at 448), S four tiles ahead of PV,
# tile j -> warpgroup j % 4, buffer j % 5: a warpgroup's next S is issued while it still works
PATCHES = [
    ("attn_fwd_sm100.cu", "constexpr int NS = 4;", "constexpr int NS = 5;"),
    ("attn_fwd_sm100.cu", "constexpr int O_COL = 256;", "constexpr int O_COL = 320;"),
    ("attn_fwd_sm100.cu", "constexpr int Q_COL = 384;", "constexpr int Q_COL = 448;"),
]
