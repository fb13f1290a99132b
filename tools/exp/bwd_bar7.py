# bisect: tail barrier id 7 instead of 1 (all three call sites)
import re
PATCHES = [("attn_bwd_sm100.cu", "named_bar_sync(1, THREADS);   // every role done with TMEM", "named_bar_sync(7, THREADS);   // every role done with TMEM"),
           ("attn_bwd_sm100.cu", "        __syncwarp();\n        named_bar_sync(1, THREADS);\n    } else {", "        __syncwarp();\n        named_bar_sync(7, THREADS);\n    } else {"),
           ("attn_bwd_sm100.cu", "        __syncwarp();\n        named_bar_sync(1, THREADS);\n    }\n}", "        __syncwarp();\n        named_bar_sync(7, THREADS);\n    }\n}")]
