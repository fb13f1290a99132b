"""NEXT-3: Load-Balanced Stochastic Length (arXiv 2602.16986 §4.1, P:109-115;
Algorithm 1) as the per-rank runtime between the data loader and the layer.

Per step each rank calls the native selection (``uh_lbsl_select``: Alg. 1 lines 4-20),
builds the kept-row list (``uh_lbsl_rows``) and gathers the kept tokens on the device
(``uh_gather_rows``).  The target l_bar is the mean of the ranks' proxy loads,
SUM-all-reduced over ``torch.distributed`` (NCCL on the B200 box, gloo in the CPU
tests) at the end of warm-up and at every recalibration (lines 22-27, reading R23).
The state here is the few scalars of Alg. 1 line 1 (l_bar, l_r, t); all arithmetic on
lengths is in the library.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch
import torch.distributed as dist

from . import uhstu as U

TRUNCATED, KEPT_BY_SL, UNSAMPLED = 0, 1, 2


@dataclass
class LbslConfig:
    T_warm: int
    T_recal: int
    gamma: float
    ell_sl: int
    seed: int = 0


class LBSL:
    """One rank's LBSL state (Alg. 1 line 1) and step (lines 2-27)."""

    def __init__(self, cfg: LbslConfig, rank: int = 0, world: int = 1, group=None):
        if not (1 < cfg.gamma < 2):
            raise ValueError("gamma must lie in (1, 2) (P:112)")
        if cfg.T_warm < 1 or cfg.T_recal < 1 or cfg.ell_sl < 1:
            raise ValueError("T_warm, T_recal, ell_sl >= 1")
        self.cfg, self.rank, self.world, self.group = cfg, rank, world, group
        self.ell_bar = 0.0
        self.ell_r = 0.0
        self.t = 0
        self.since_reset = 0

    def _allreduce_sum(self, v: float) -> float:
        if self.world == 1 or not dist.is_available() or not dist.is_initialized():
            return v
        dev = "cuda" if dist.get_backend(self.group) == "nccl" else "cpu"
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
        return float(t.item())

    def select(self, lengths):
        """Lines 2-27 for this rank: returns (decision[b], new_len[b]) and advances t."""
        c = self.cfg
        t = self.t + 1
        dec, new, proxy = U.lbsl_select(lengths, c.ell_sl, c.gamma, self.ell_bar, t > c.T_warm, c.seed, self.rank, t)
        self.ell_r += proxy                                     # line 5
        self.since_reset += 1
        if t == c.T_warm or (t > c.T_warm and t % c.T_recal == 0):   # lines 22-27 (R23)
            self.ell_bar = self._allreduce_sum(self.ell_r) / (self.world * self.since_reset)
            self.ell_r = 0.0
            self.since_reset = 0
        self.t = t
        return dec, new

    def apply(self, jag: U.JaggedBatch, x: torch.Tensor, device: Optional[str] = None):
        """One LBSL step on a resident jagged batch: decisions on the host, then the kept
        rows of x gathered on the device.  Returns (new JaggedBatch, x', decision)."""
        dec, new = self.select(jag.lengths)
        rows, new_off = U.lbsl_rows(jag.host, dec, new, self.cfg.seed, self.rank, self.t)
        rows_dev = torch.from_numpy(rows).to(x.device, non_blocking=False)
        y = U.gather_rows(rows_dev, x)
        return U.JaggedBatch(new_off, device=device or str(x.device)), y, dec
