# GEMM: three epilogue warpgroups for the single-CTA 256-wide bf16-out tiles (512 threads, 3 stages)
import os
H = os.path.dirname(os.path.abspath(__file__))
PATCHES = [("gemm_sm100.cuh", None, open(os.path.join(H, "gemm3wg.cuh.txt")).read()),
           ("gemm.cu", None, open(os.path.join(H, "gemm3wg_gemm.cu.txt")).read())]
