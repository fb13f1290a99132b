# forward with three S buffers (LAG 2)
PATCHES = [("attn_fwd_sm100.cu", "constexpr int NS = 4;", "constexpr int NS = 3;")]
