# bisect: no setmaxnreg, the old __syncthreads tail
PATCHES = [("attn_bwd_sm100.cu", 'asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\\n" ::"n"(REG_CTRL));', ''),
           ("attn_bwd_sm100.cu", 'asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\\n" ::"n"(REG_PDS));', ''),
           ("attn_bwd_sm100.cu", 'asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\\n" ::"n"(REG_DQ));', ''),
           ("attn_bwd_sm100.cu", "    named_bar_sync(1, THREADS);   // every role done with TMEM\n    if (warp == 2) tmem_dealloc<512>(tmem);", ""),
           ("attn_bwd_sm100.cu", "        __syncwarp();\n        named_bar_sync(1, THREADS);\n    } else {", "    } else {"),
           ("attn_bwd_sm100.cu", "        __syncwarp();\n        named_bar_sync(1, THREADS);\n    }\n}", "    }\n    __syncthreads();\n    if (warp == 2) tmem_dealloc<512>(tmem);\n}")]
