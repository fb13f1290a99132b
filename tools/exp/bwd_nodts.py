# backward: skip the time-bias gradient accumulation (cost of the d time_bias runs)
PATCHES = [("attn_bwd_sm100.cu", "                if (a.dts) {   // runs of equal time bucket", "                if (false) {   // runs of equal time bucket")]
