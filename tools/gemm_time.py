"""Time the projection GEMM (test hook) for the layer's shapes and operand majors (CUDA events)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2602_16986_b200 import uhstu as U  # noqa: E402
if os.environ.get("UH_LIB"):   # experiment builds (tools/build_exp.py)
    U.LIB_PATH = os.path.join(ROOT, "paper_2602_16986_b200", "lib", os.environ["UH_LIB"])


def t(fn, it=10):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(it):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / it


T, d = 262144, 512
A = torch.randn(T, d, device="cuda").to(torch.bfloat16)
W = (torch.randn(d, 4 * d, device="cuda") / d ** 0.5).to(torch.bfloat16)     # [K, N] (MN-major B)
Wt = W.t().contiguous()                                                       # [N, K] (K-major B)
bias = torch.zeros(4 * d, device="cuda")
o0 = torch.empty(T, 4 * d, device="cuda", dtype=torch.bfloat16)
o1 = torch.empty_like(o0)
PAIR = int(os.environ.get("PAIR", "0"))
tag = f"pair={PAIR}"
for name, B, bmn in (("B MN-major [K,N]", W, True), ("B K-major [N,K]", Wt, False)):
    for outs in (1, 2):
        ms = t(lambda: U.test_gemm(A, B, False, bmn, 1, T, 4 * d, d, bias=bias, out0=o0, out1=o1 if outs == 2 else None, cta_pair=PAIR))
        print(f"{tag} f1 SiLU {name} outputs={outs}: {ms:.3f} ms  {2 * T * d * 4 * d / ms / 1e9:.0f} TFLOP/s", flush=True)
# f2 (bias + residual epilogue), dY = dOut W2^T (K-major B), dx^ = dH W1^T (K = 4d, K-major B)
W2 = (torch.randn(d, d, device="cuda") / d ** 0.5).to(torch.bfloat16)
b2 = torch.zeros(d, device="cuda")
R = torch.randn(T, d, device="cuda").to(torch.bfloat16)
O = torch.empty(T, d, device="cuda", dtype=torch.bfloat16)
ms = t(lambda: U.test_gemm(A, W2, False, True, 0, T, d, d, bias=b2, resid=R, out0=O, cta_pair=PAIR))
print(f"{tag} f2 bias+resid B MN-major: {ms:.3f} ms  {2 * T * d * d / ms / 1e9:.0f} TFLOP/s", flush=True)
ms = t(lambda: U.test_gemm(A, W2, False, False, 0, T, d, d, out0=O))
print(f"{tag} dY B K-major: {ms:.3f} ms  {2 * T * d * d / ms / 1e9:.0f} TFLOP/s", flush=True)
ms = t(lambda: U.test_gemm(o0, W, False, False, 0, T, d, 4 * d, out0=O))
print(f"{tag} dx^ K=4d B K-major: {ms:.3f} ms  {2 * T * d * 4 * d / ms / 1e9:.0f} TFLOP/s", flush=True)
