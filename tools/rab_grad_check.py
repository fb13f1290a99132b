"""Relative errors of d pos_bias / d time_bias (and dQ, dK, dV) of the bf16 attention backward
against the oracle at the cfg3 shape on a few full-length sequences.  usage: rab_grad_check.py [B]"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle as O  # noqa: E402
from paper_2602_16986_b200 import synth  # noqa: E402
from paper_2602_16986_b200 import uhstu as U  # noqa: E402

if os.environ.get("UH_LIB"):
    U.LIB_PATH = os.path.join(ROOT, "paper_2602_16986_b200", "lib", os.environ["UH_LIB"])


def rel(g, r):
    return float(np.max(np.abs(np.asarray(g, np.float64) - r)) / max(np.max(np.abs(r)), 1e-300))


B = int(sys.argv[1]) if len(sys.argv) > 1 else 2
for P in (16384, 128):
    cfg = synth.Config("chk", [16384] * B, H=4, dh=128, K1=1024, K2=128, N=16384.0, seed=3, pos_len=P)
    q, k, v, dA = synth.attn_inputs(cfg)
    pos, ts = synth.rab_tables(cfg)
    t = synth.timestamps(cfg.seed, cfg.lengths)
    d = cfg.d
    buf = torch.empty(cfg.T, 4 * d, dtype=torch.bfloat16, device="cuda")
    for j, a in ((1, v), (2, q), (3, k)):
        buf[:, j * d:(j + 1) * d] = torch.from_numpy(a).to("cuda", torch.bfloat16)
    attn = U.Attn(4, 128, 1.0, 16384.0, torch.from_numpy(pos).cuda(), torch.from_numpy(ts).cuda(),
                  torch.from_numpy(t).cuda())
    jag = U.JaggedBatch(cfg.offsets())
    m = U.mask(1024, 128)
    Q, K, V = buf[:, 2 * d:3 * d], buf[:, 3 * d:], buf[:, d:2 * d]
    dq, dk, dv, dpos, dts = U.attn_bwd(jag, m, attn, Q, K, V, torch.from_numpy(dA).to("cuda", torch.bfloat16))
    torch.cuda.synchronize()
    spec = O.AttnSpec(K1=1024, K2=128, alpha=1.0, N=16384.0, pos_w=pos, ts_w=ts, timestamps=t)
    ref = O.attention_backward(cfg.offsets(), 4, 128, q, k, v, dA, spec)
    f = lambda x: x.float().cpu().numpy()
    print(f"P={P} B={B}: dQ {rel(f(dq), ref[0]):.2e} dK {rel(f(dk), ref[1]):.2e} dV {rel(f(dv), ref[2]):.2e} "
          f"dpos {rel(f(dpos), ref[3]):.2e} dts {rel(f(dts), ref[4]):.2e}", flush=True)
    r4 = ref[4]
    print("   dts ref:", np.array2string(r4, precision=3, max_line_width=200))
    print("   dts gpu:", np.array2string(f(dts), precision=3, max_line_width=200))
