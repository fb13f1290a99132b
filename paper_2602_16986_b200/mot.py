"""NEXT-4: Mixture of Transducers over the C ABI (no arithmetic here: every step is a library call).

P:202 (§4.3) "MoT processes multiple distinct input sequences through separate transducers and
subsequently fuses the learned user embeddings"; App. A P:390-392 runs two of them (consumption
and engagement sequences, the "10k C-seq and 3k E-seq" row of the MoT table).  Each
branch is a ``dist.Stack`` (its own layers, depth and mask, reading R30) on its own jagged batch
of the same users; ``uh_mot_fuse_fwd`` / ``uh_mot_fuse_bwd`` (include/uhstu_mot.h) gather the
candidate rows (the last ``n_cand`` of every sequence, R29), concatenate them and project to d
(R28).  The fusion's fp32 gradients live in their own flat bucket, all-reduced like a layer's.
"""
from __future__ import annotations

from typing import List, Optional, Sequence

import torch

from . import uhstu as U
from .dist import GradBucket, Stack

FUSE_NAMES = ("w_f", "b_f")


class MoT:
    def __init__(self, branches: Sequence[Stack], n_cand: int, w_f: torch.Tensor, b_f: Optional[torch.Tensor]):
        self.branches = list(branches)
        self.n_cand = int(n_cand)
        self.w_f, self.b_f = w_f, b_f
        d = w_f.shape[1]
        dev = w_f.device
        self.bucket = GradBucket(dict(w_f=tuple(w_f.shape), b_f=None if b_f is None else tuple(b_f.shape)), dev,
                                 names=FUSE_NAMES)
        self.jags = [b.jag for b in self.branches]
        self.states: List[torch.Tensor] = []
        C = self.jags[0].B * self.n_cand
        dt = w_f.dtype
        self.e = torch.empty(C, d, dtype=dt, device=dev)
        self.dxs = [torch.empty(j.T, d, dtype=dt, device=dev) for j in self.jags]
        self.ws = None

    def _ws(self, xs):
        if self.ws is None:
            self.ws = U._ws(U.mot_workspace_bytes(self.jags, xs, self.n_cand, True), xs[0].device)
        return self.ws

    def forward(self, xs: Sequence[torch.Tensor]) -> torch.Tensor:
        """Every branch's stack, then E = concat_k X_k[candidates] W_f + b_f: [B n_cand, d]."""
        self.states = [br.forward(x) for br, x in zip(self.branches, xs)]
        return U.mot_fuse_fwd(self.jags, self.states, self.n_cand, self.w_f, self.b_f, out=self.e,
                              ws=self._ws(self.states))

    def backward(self, xs: Sequence[torch.Tensor], de: torch.Tensor, group=None):
        """After forward(xs): the fusion backward (its gradients into self.bucket, all-reduced
        asynchronously), then each branch's stack backward seeded with its candidate-row
        gradient.  Returns (dxs, handles)."""
        U.mot_fuse_bwd(self.jags, self.states, self.n_cand, self.w_f, de, self.bucket.views["w_f"],
                       self.bucket.views["b_f"], dxs=self.dxs, ws=self._ws(self.states))
        handles = []
        hd = self.bucket.allreduce_(group, async_op=True)
        if hd is not None:
            handles.append(hd)
        dxs = []
        for br, x, g in zip(self.branches, xs, self.dxs):
            dx, h = br.backward(x, g, group)
            dxs.append(dx)
            handles += h
        return dxs, handles
