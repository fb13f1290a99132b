"""Profiling driver: one cfg3-shaped layer fwd+bwd (and attention alone) at a reduced
batch so ncu --set full replays stay short.  Usage: python tools/prof_layer.py [B] [iters]"""
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


def main():
    B = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    cfg = synth.config("cfg3")
    lengths = [16384] * B
    dev = torch.device("cuda")
    x, dout = synth.layer_inputs(cfg, lengths=lengths)
    t = synth.timestamps(cfg.seed, lengths)
    pos, ts = synth.rab_tables(cfg)
    p = synth.layer_params(cfg.d, cfg.seed)
    f = lambda a: torch.from_numpy(a).to(dev)
    b = lambda a: torch.from_numpy(a).to(dev, torch.bfloat16)
    prm = U.Params(f(p["ln1_w"]), f(p["ln1_b"]), b(p["w1"]), f(p["ln2_w"]), f(p["ln2_b"]), b(p["w2"]), f(p["b1"]),
                   f(p["b2"]))
    jag = U.JaggedBatch.from_lengths(lengths)
    attn = U.Attn(cfg.H, cfg.dh, 1.0, float(cfg.N), f(pos), f(ts), f(t))
    m = U.mask(cfg.K1, cfg.K2)
    X, D = b(x), b(dout)
    for _ in range(iters):
        out, saved = U.layer_fwd(jag, m, prm, attn, X)
        dx, g = U.layer_bwd(jag, m, prm, attn, X, saved, D)
    torch.cuda.synchronize()
    print("ok", float(out.float().abs().mean()), float(dx.float().abs().mean()))


if __name__ == "__main__":
    main()
