"""Small ragged cases for compute-sanitizer (memcheck / racecheck / synccheck): the tcgen05
attention forward and backward, the layer forward and backward (GEMMs, norm kernels) and a
jagged gather, each on a batch that mixes sub-tile, tile-straddling and empty sequences.
usage: compute-sanitizer --tool memcheck python tools/sanitize_case.py"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2602_16986_b200 import synth  # noqa: E402
from paper_2602_16986_b200 import uhstu as U  # noqa: E402


def main():
    lengths = [17, 0, 40, 64, 129, 1, 300]
    for K1, K2 in ((16, 2), (127, 129), (synth.WINDOW_FULL, 0)):
        cfg = synth.Config("san", lengths, H=2, dh=128, K1=K1, K2=K2, N=300.0, seed=1, pos_len=200, ts_len=32)
        q, k, v, dA = (torch.from_numpy(a).cuda().to(torch.bfloat16) for a in synth.attn_inputs(cfg))
        pos, ts = synth.rab_tables(cfg)
        t = synth.timestamps(1, lengths)
        attn = U.Attn(2, 128, 1.0, 300.0, torch.from_numpy(pos).cuda(), torch.from_numpy(ts).cuda(),
                      torch.from_numpy(t).cuda())
        jag = U.JaggedBatch.from_lengths(lengths)
        m = U.mask(K1, K2)
        A = U.attn_fwd(jag, m, attn, q, k, v)
        dq, dk, dv, dpos, dts = U.attn_bwd(jag, m, attn, q, k, v, dA)
        torch.cuda.synchronize()
        print("attn", K1, K2, float(A.float().abs().sum()), float(dq.float().abs().sum()), flush=True)
    # one layer fwd + bwd (LN, f1 GEMM + SiLU, attention, gated norm, f2 + residual; the remat backward)
    cfg = synth.Config("san", lengths, H=2, dh=128, K1=16, K2=2, N=300.0, seed=2, pos_len=200, ts_len=32)
    p = synth.layer_params(cfg.d, 2)
    x, dout = synth.layer_inputs(cfg)
    f = lambda a: torch.from_numpy(a).cuda()
    b = lambda a: torch.from_numpy(a).cuda().to(torch.bfloat16)
    prm = U.Params(f(p["ln1_w"]), f(p["ln1_b"]), b(p["w1"]), f(p["ln2_w"]), f(p["ln2_b"]), b(p["w2"]), f(p["b1"]),
                   f(p["b2"]))
    pos, ts = synth.rab_tables(cfg)
    attn = U.Attn(2, 128, 1.0, 300.0, f(pos), f(ts), f(synth.timestamps(2, lengths)))
    jag = U.JaggedBatch.from_lengths(lengths)
    m = U.mask(16, 2)
    X, D = b(x), b(dout)
    out, saved = U.layer_fwd(jag, m, prm, attn, X)
    dx, g = U.layer_bwd(jag, m, prm, attn, X, saved, D)
    y, _ = U.jagged_gather(jag, [6, 2, 0], X)
    torch.cuda.synchronize()
    print("layer", float(out.float().abs().sum()), float(dx.float().abs().sum()), float(y.float().abs().sum()),
          flush=True)


if __name__ == "__main__":
    main()
