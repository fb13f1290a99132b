# backward: no setmaxnreg (640 threads at the launch register count)
PATCHES = [("attn_bwd_sm100.cu", 'asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\\n" ::"n"(REG_CTRL));', ''),
           ("attn_bwd_sm100.cu", 'asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\\n" ::"n"(REG_PDS));', ''),
           ("attn_bwd_sm100.cu", 'asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\\n" ::"n"(REG_DQ));', '')]
