"""Helpers shared by the GPU parity tests: seeded inputs (synth), the oracle side
and the CUDA side (through the C-ABI binding) on identical values."""
import numpy as np
import torch

import oracle as O
from paper_2602_16986_b200 import synth
from paper_2602_16986_b200 import uhstu as U


def rel_inf(gpu, ref):
    """Per-tensor infinity-norm relative error (R15)."""
    g = np.asarray(gpu, np.float64)
    r = np.asarray(ref, np.float64)
    den = np.max(np.abs(r)) if r.size else 0.0
    if den == 0.0:
        return float(np.max(np.abs(g))) if g.size else 0.0
    return float(np.max(np.abs(g - r)) / den)


def tdt(dtype):
    return torch.bfloat16 if dtype == U.BF16 else torch.float32


def to_dev(a, dtype):
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda", tdt(dtype))


def to_np(t):
    return t.detach().float().cpu().numpy()


def oracle_k1(K1):
    return O.FULL if K1 >= synth.WINDOW_FULL else K1


class AttnCase:
    def __init__(self, lengths, H=2, dh=128, K1=16, K2=2, N=64.0, rab=True, seed=0, P=0, NB=32, alpha=1.0):
        self.cfg = synth.Config("case", list(lengths), H=H, dh=dh, K1=K1, K2=K2, N=N, seed=seed, pos_len=P,
                                ts_len=NB, alpha=alpha)
        self.q, self.k, self.v, self.dA = synth.attn_inputs(self.cfg)
        self.pos, self.ts = synth.rab_tables(self.cfg) if rab else (None, None)
        self.t = synth.timestamps(seed, lengths) if rab else None
        self.alpha = alpha

    def spec(self):
        c = self.cfg
        return O.AttnSpec(K1=oracle_k1(c.K1), K2=c.K2, alpha=self.alpha, N=c.N, pos_w=self.pos, ts_w=self.ts,
                          timestamps=self.t)

    def desc(self):
        c = self.cfg
        return U.Attn(c.H, c.dh, self.alpha, float(c.N),
                      None if self.pos is None else torch.from_numpy(self.pos).cuda(),
                      None if self.ts is None else torch.from_numpy(self.ts).cuda(),
                      None if self.t is None else torch.from_numpy(self.t).cuda())

    def mask(self):
        return U.mask(self.cfg.K1, self.cfg.K2)

    def jag(self):
        return U.JaggedBatch(self.cfg.offsets())

    def fused_qkv(self, dtype):
        """Q, K, V as column views of one [T, 4d] buffer laid out U|V|Q|K like the layer's."""
        d = self.cfg.d
        buf = torch.zeros(self.cfg.T, 4 * d, dtype=tdt(dtype), device="cuda")
        buf[:, d:2 * d] = to_dev(self.v, dtype)
        buf[:, 2 * d:3 * d] = to_dev(self.q, dtype)
        buf[:, 3 * d:] = to_dev(self.k, dtype)
        return buf, buf[:, 2 * d:3 * d], buf[:, 3 * d:], buf[:, d:2 * d]
