# measurement only (wrong d time_bias): the P/dS warps skip the d time_bias runs
PATCHES = [("attn_bwd_sm100.cu", "if (a.dts) {   // runs of equal time bucket", "if (false) {   // runs of equal time bucket")]
