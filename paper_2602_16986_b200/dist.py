"""Data-parallel plumbing of the hot path: every rank computes the same
token-balanced LPT assignment of the global jagged batch (``uh_partition_lpt``, host
C++), processes its own sequences, and the layer's fp32 parameter gradients are SUM
all-reduced in one flat bucket (NCCL over NVLink/NVSwitch on the B200 box; gloo in the
CPU tests).  Parameter gradients are sums over tokens, so the all-reduced result equals
the single-process gradient of the whole batch up to fp32 reassociation.
"""
from __future__ import annotations

from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np
import torch
import torch.distributed as dist

from . import uhstu as U

GRAD_NAMES = ("ln1_w", "ln1_b", "w1", "b1", "ln2_w", "ln2_b", "w2", "b2", "pos_bias", "time_bias")


def shard(lengths: Sequence[int], world: int, rank: int, m: U.Mask, d: int, num_heads: int
          ) -> Tuple[List[int], List[int], np.ndarray]:
    """This rank's global sequence ids (ascending), their lengths, and all ranks' costs."""
    owner, cost = U.partition_lpt(lengths, world, m, d, num_heads)
    ids = [i for i in range(len(lengths)) if owner[i] == rank]
    return ids, [int(lengths[i]) for i in ids], cost


class GradBucket:
    """One flat fp32 buffer holding every parameter gradient; each view is 16-byte aligned
    (the C-ABI's alignment contract) and the whole bucket is one all-reduce."""

    def __init__(self, shapes: Dict[str, Optional[Tuple[int, ...]]], device):
        n = 0
        self.offsets = {}
        for k in GRAD_NAMES:
            s = shapes.get(k)
            if s is None:
                continue
            numel = int(np.prod(s))
            self.offsets[k] = (n, s)
            n += (numel + 3) // 4 * 4
        self.flat = torch.zeros(max(n, 4), dtype=torch.float32, device=device)
        self.views = {k: None for k in GRAD_NAMES}
        for k, (o, s) in self.offsets.items():
            self.views[k] = self.flat[o:o + int(np.prod(s))].view(s)

    @staticmethod
    def for_layer(prm: U.Params, attn: U.Attn, device) -> "GradBucket":
        shp = lambda t: None if t is None else tuple(t.shape)
        return GradBucket(dict(ln1_w=shp(prm.ln1_w), ln1_b=shp(prm.ln1_b), w1=shp(prm.w1), b1=shp(prm.b1),
                               ln2_w=shp(prm.ln2_w), ln2_b=shp(prm.ln2_b), w2=shp(prm.w2), b2=shp(prm.b2),
                               pos_bias=shp(attn.pos_bias), time_bias=shp(attn.time_bias)), device)

    def zero_(self):
        self.flat.zero_()

    def allreduce_(self, group=None, async_op: bool = False):
        """SUM over ranks (the weight-gradient exchange of synchronous DP)."""
        if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
            return None
        return dist.all_reduce(self.flat, op=dist.ReduceOp.SUM, group=group, async_op=async_op)


def layer_step(jag: U.JaggedBatch, m: U.Mask, prm: U.Params, attn: U.Attn, x: torch.Tensor, dout: torch.Tensor,
               bucket: GradBucket, saved: Optional[U.Saved] = None, out=None, dx=None, ws_f=None, ws_b=None,
               group=None):
    """One data-parallel training step of one HSTU layer on this rank's shard: forward,
    rematerialising backward (gradients into the bucket), then the bucket all-reduce."""
    out, saved = U.layer_fwd(jag, m, prm, attn, x, out=out, ws=ws_f, saved=saved)
    dx, _ = U.layer_bwd(jag, m, prm, attn, x, saved, dout, grads=bucket.views, dx=dx, ws=ws_b)
    bucket.allreduce_(group)
    return out, dx
