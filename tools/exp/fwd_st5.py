# forward: 5 (K,V) stages
PATCHES = [("attn_fwd_sm100.cu", "constexpr int STAGES = 4;", "constexpr int STAGES = 5;")]
