# backward: accurate tanhf in the P/dS epilogue (precision check of the rab gradients)
PATCHES = [("attn_bwd_sm100.cu", "const uint64_t T = f2_pack(tanh_approx(hx[2 * c]), tanh_approx(hx[2 * c + 1]));",
            "const uint64_t T = f2_pack(tanhf(hx[2 * c]), tanhf(hx[2 * c + 1]));")]
