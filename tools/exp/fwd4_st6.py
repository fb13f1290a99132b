# fwd (4 warpgroups): six (K, V) stages (the K of tile j loads once PV(j - 6) has completed)
PATCHES = [("attn_fwd_sm100.cu", "constexpr int STAGES = 5;", "constexpr int STAGES = 6;")]
