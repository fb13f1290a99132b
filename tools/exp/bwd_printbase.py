# backward: print the dynamic shared memory base (debugging)
PATCHES = [("attn_bwd_sm100.cu", "    if (smem_u32(smem_raw) & 1023) __trap();",
            "    if (blockIdx.x == 0 && threadIdx.x == 0) printf(\"smem base 0x%x\\n\", smem_u32(smem_raw));")]
