"""One launch each of the cfg3 projections for ncu (T = 262144, d = 512): f1 bf16 (SiLU epilogue),
f1 fp8, f2 bf16 (+ residual), f2 fp8.  usage: ncu ... python tools/gemm_once.py"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2602_16986_b200 import uhstu as U  # noqa: E402

T, d = 262144, 512
dev = "cuda"
A = torch.randn(T, d, device=dev).to(torch.bfloat16)
W1 = (torch.randn(d, 4 * d, device=dev) / d ** 0.5).to(torch.bfloat16)
W2 = (torch.randn(d, d, device=dev) / d ** 0.5).to(torch.bfloat16)
b1 = torch.zeros(4 * d, device=dev); b2 = torch.zeros(d, device=dev)
o1 = torch.empty(T, 4 * d, device=dev, dtype=torch.bfloat16)
o2 = torch.empty(T, d, device=dev, dtype=torch.bfloat16)
w = torch.ones(d, device=dev); bb = torch.zeros(d, device=dev)
qa, sa = U.ln_fwd_fp8(A, w, bb)
q1, s1 = U.quant_weight_fp8(W1)
q2, s2 = U.quant_weight_fp8(W2)
torch.cuda.synchronize()
U.test_gemm(A, W1, False, True, 1, T, 4 * d, d, bias=b1, out0=o1)
U.gemm_fp8(qa, sa, q1, s1, 1, bias=b1, out=o1)
U.test_gemm(A, W2, False, True, 0, T, d, d, bias=b2, resid=A, out0=o2)
U.gemm_fp8(qa, sa, q2, s2, 0, bias=b2, resid=A, out=o2)
torch.cuda.synchronize()
