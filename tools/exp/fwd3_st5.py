# fwd (3 warpgroups): five (K, V) stages
PATCHES = [("attn_fwd_sm100.cu", "constexpr int STAGES = 4;", "constexpr int STAGES = 5;")]
