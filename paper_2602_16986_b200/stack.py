"""Multi-layer orchestration over the C ABI (no arithmetic here: every step is a library call).

``forward_truncated`` is SURVEY §8(f) NEXT-1, the inference schedule of cfg5: the first
``n_full`` layers run on the whole jagged sequences under the semi-local mask (SLA,
P:137-147); then the latest ``l_keep`` tokens of every sequence are gathered
(``uh_jagged_slice_latest`` — "simply truncating the latest UIH segment") and
the remaining layers run full-causal on them ("attention truncation").
Timestamps (time-bias rab) are sliced with the same row map.
"""
from __future__ import annotations

from dataclasses import dataclass, replace
from typing import List, Optional

import torch

from . import uhstu as U


@dataclass
class Layer:
    params: U.Params
    attn: U.Attn          # timestamps (if any) are those of the full sequences
    mask: U.Mask


def forward_truncated(jag: U.JaggedBatch, x: torch.Tensor, layers: List[Layer], n_full: int, l_keep: int,
                      norm_n_truncated: Optional[float] = None, ws: Optional[torch.Tensor] = None,
                      bufs: Optional[List[torch.Tensor]] = None):
    """Forward-only stack (inference, nothing saved).  Returns (out, jag_out): the output rows of
    the truncated segment and its jagged batch (the whole batch if n_full == len(layers)).
    ``ws`` (one layer workspace) and ``bufs`` (two [T, d] ping-pong outputs) may be passed so a
    batch that fills the GPU allocates nothing per layer."""
    h = x
    for i, lay in enumerate(layers[:n_full]):
        out = bufs[i % 2] if bufs is not None else None
        h, _ = U.layer_fwd(jag, lay.mask, lay.params, lay.attn, h, save=False, out=out, ws=ws)
    if n_full == len(layers):
        return h, jag
    nxt = None
    if bufs is not None:   # h lives in bufs[(n_full - 1) % 2]; the truncated rows go to the other one
        n_keep = int(sum(min(int(L), l_keep) for L in jag.lengths))
        nxt = [bufs[n_full % 2][:n_keep], bufs[(n_full - 1) % 2][:n_keep]]
    h, jt = U.jagged_slice_latest(jag, l_keep, h, out=nxt[0] if nxt else None)
    ts_cache = {}
    for i, lay in enumerate(layers[n_full:]):
        attn = lay.attn
        if attn.timestamps is not None:
            key = attn.timestamps.data_ptr()
            if key not in ts_cache:
                t2, _ = U.jagged_slice_latest(jag, l_keep, attn.timestamps.view(-1, 1))
                ts_cache[key] = t2.view(-1)
            attn = replace(attn, timestamps=ts_cache[key])
        if norm_n_truncated is not None:
            attn = replace(attn, norm_n=float(norm_n_truncated))
        h, _ = U.layer_fwd(jt, lay.mask, lay.params, attn, h, save=False, out=nxt[(i + 1) % 2] if nxt else None,
                           ws=ws)
    return h, jt
