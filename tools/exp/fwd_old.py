# round-1 forward kernel (git HEAD~ of attn_fwd_sm100.cu) for A/B timing
import os
PATCHES = [("attn_fwd_sm100.cu", None, open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "old_fwd.cu.txt")).read())]
