"""NEXT-2 timing at cfg3 widths (T = 262144, d = 512): FP8 vs bf16 projections, the fused
norm+quant kernels, and the whole layer forward (inference) both ways.  CUDA events."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2602_16986_b200 import synth  # noqa: E402
from paper_2602_16986_b200 import uhstu as U  # noqa: E402
if os.environ.get("UH_LIB"):   # experiment builds (tools/build_exp.py)
    U.LIB_PATH = os.path.join(ROOT, "paper_2602_16986_b200", "lib", os.environ["UH_LIB"])


def t(fn, it=20):
    for _ in range(3):
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
f1 = 2 * T * d * 4 * d
f2 = 2 * T * d * d
ms = t(lambda: U.test_gemm(A, W1, False, True, 1, T, 4 * d, d, bias=b1, out0=o1))
print(f"f1 bf16 SiLU: {ms:.3f} ms {f1 / ms / 1e9:.0f} TFLOP/s", flush=True)
ms = t(lambda: U.gemm_fp8(qa, sa, q1, s1, 1, bias=b1, out=o1))
print(f"f1 fp8  SiLU: {ms:.3f} ms {f1 / ms / 1e9:.0f} TFLOP/s", flush=True)
ms = t(lambda: U.test_gemm(A, W2, False, True, 0, T, d, d, bias=b2, resid=A, out0=o2))
print(f"f2 bf16 +resid: {ms:.3f} ms {f2 / ms / 1e9:.0f} TFLOP/s", flush=True)
ms = t(lambda: U.gemm_fp8(qa, sa, q2, s2, 0, bias=b2, resid=A, out=o2))
print(f"f2 fp8  +resid: {ms:.3f} ms {f2 / ms / 1e9:.0f} TFLOP/s", flush=True)
ms = t(lambda: U.ln_fwd_fp8(A, w, bb, q=qa, scale=sa))
print(f"ln_fwd_fp8: {ms * 1e3:.1f} us {(T * d * 3 + T * 4) / ms / 1e6:.0f} GB/s", flush=True)
ms = t(lambda: U.gated_norm_fwd_fp8(A, o1[:, :d], w, bb, q=qa, scale=sa))
print(f"gated_norm_fwd_fp8: {ms * 1e3:.1f} us {(T * d * 5 + T * 4) / ms / 1e6:.0f} GB/s", flush=True)
ms = t(lambda: U.quant_weight_fp8(W1))
print(f"quant_weight_fp8 W1: {ms * 1e3:.1f} us", flush=True)

cfg = synth.config("cfg3")
p = synth.layer_params(cfg.d, cfg.seed)
x, _ = synth.layer_inputs(cfg)
pos, ts = synth.rab_tables(cfg)
tt = synth.timestamps(cfg.seed, cfg.lengths)
f = lambda a: torch.from_numpy(a).cuda()
b = lambda a: torch.from_numpy(a).to("cuda", torch.bfloat16)
prm = U.Params(f(p["ln1_w"]), f(p["ln1_b"]), b(p["w1"]), f(p["ln2_w"]), f(p["ln2_b"]), b(p["w2"]),
               f(p["b1"]), f(p["b2"]))
attn = U.Attn(cfg.H, cfg.dh, 1.0, float(cfg.N), f(pos), f(ts), f(tt))
jag = U.JaggedBatch(cfg.offsets())
m = U.mask(cfg.K1, cfg.K2)
X = b(x)
out = torch.empty_like(X)
ws = torch.empty(U.layer_workspace_bytes(jag, m, prm, attn, U.BF16, False), dtype=torch.uint8, device=dev)
qw = U.quant_layer_weights(prm)
ms_b = t(lambda: U.layer_fwd(jag, m, prm, attn, X, save=False, out=out, ws=ws), it=10)
ms_f = t(lambda: U.layer_fwd_fp8(jag, m, prm, attn, X, qw, save=False, out=out, ws=ws), it=10)
print(f"cfg3 layer fwd (inference): bf16 {ms_b:.3f} ms ({T / ms_b / 1e3:.2f} M tok/s), "
      f"fp8 projections {ms_f:.3f} ms ({T / ms_f / 1e3:.2f} M tok/s)", flush=True)
