# fwd (3 warpgroups): four S buffers (S three tiles ahead of PV), tile j -> warpgroup j % 3
PATCHES = [("attn_fwd_sm100.cu", "constexpr int NS = 3;", "constexpr int NS = 4;")]
