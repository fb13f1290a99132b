"""ORACLE — test infrastructure only (NEXT-4: Mixture of Transducers).

Plain fp64 CPU reference of SURVEY §8(f) NEXT-4.  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import it; the CUDA path
(``paper_2602_16986_b200``) never imports it and shares no code with it.

What the paper fixes (PAPER.md, ``P:n`` = line n):
* P:202 (§4.3) "MoT processes multiple distinct input sequences through separate transducers
  and subsequently fuses the learned user embeddings"; "the model can assign deeper layers and
  greater capacity to high-value sequences".
* P:390-392 (App. A) "two specialized HSTU modules: one for engagement events and one for
  consumption events" (E-seq / C-seq of the MoT table).
* P:74 / P:104: the model scores candidates x_j, which sit in the sequence (their action
  embeddings masked to zero).

Readings (where the paper is silent):
* R28  the fusion is the concatenation of the branches' outputs at the candidate positions
       followed by one linear projection [K d -> d] with bias (SPEC S:350-358's reading; the
       paper does not name the fusion operator).
* R29  candidates are the last ``n_cand`` rows of every sequence of every branch; every branch
       holds the same B users in the same order and the same ``n_cand`` (SPEC: "every branch
       contains the same candidate items at its tail"); a sequence shorter than ``n_cand`` or
       a branch with another user count is an error.
* R30  a branch is a plain stack of HSTU layers (``oracle.layer_forward``) with its own
       parameters, depth and mask ("deeper layers and greater capacity").

The backward is the exact chain rule of ``mot_forward`` for the loss sum(dE * E).
Every step is a numpy primitive or a call into ``oracle.py``; nothing is fused or reordered.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Sequence, Tuple

import numpy as np

import oracle as O


@dataclass
class Branch:
    """One transducer: its jagged inputs and its layer list [(LayerParams, H, AttnSpec)]."""
    x: np.ndarray                 # [T_k, d]
    offsets: np.ndarray           # int32 [B + 1]
    layers: Sequence[Tuple[O.LayerParams, int, O.AttnSpec]]


def candidate_rows(offsets, n_cand: int) -> np.ndarray:
    """R29: rows offsets[b+1] - n_cand + j of every sequence b, in (b, j) order."""
    offsets = np.asarray(offsets, dtype=np.int64)
    if n_cand <= 0:
        raise ValueError("n_cand must be positive")
    rows = []
    for b in range(len(offsets) - 1):
        L = int(offsets[b + 1] - offsets[b])
        if L < n_cand:
            raise ValueError(f"sequence {b} has {L} rows < n_cand = {n_cand}")
        for j in range(n_cand):
            rows.append(int(offsets[b + 1]) - n_cand + j)
    return np.asarray(rows, dtype=np.int64)


def branch_forward(br: Branch):
    """R30: the branch's layers in order on its full sequences.  Returns (out, caches)."""
    h = np.asarray(br.x, dtype=np.float64)
    caches = []
    for prm, H, spec in br.layers:
        h, c = O.layer_forward(h, br.offsets, prm, H, spec)
        caches.append(c)
    return h, caches


def branch_backward(dout, br: Branch, caches):
    """Chain rule through the branch's layers in reverse.  Returns (dx, [grads per layer])."""
    g = np.asarray(dout, dtype=np.float64)
    grads = [None] * len(br.layers)
    for i in range(len(br.layers) - 1, -1, -1):
        prm, H, spec = br.layers[i]
        g, grads[i] = O.layer_backward(g, br.offsets, prm, H, spec, cache=caches[i])
    return g, grads


def mot_forward(branches: List[Branch], n_cand: int, Wf, bf):
    """E = concat_k(out_k[cand rows]) Wf + bf  (R28), E: [B n_cand, d].  Returns (E, cache)."""
    if not branches:
        raise ValueError("MoT needs at least one branch")
    B = len(branches[0].offsets) - 1
    for br in branches:
        if len(br.offsets) - 1 != B:
            raise ValueError("every branch must hold the same users (R29)")
    outs, caches, rows, Z = [], [], [], []
    for br in branches:
        out, c = branch_forward(br)
        r = candidate_rows(br.offsets, n_cand)
        outs.append(out)
        caches.append(c)
        rows.append(r)
        Z.append(out[r])                                     # the branch's user embeddings per candidate
    Zcat = np.concatenate(Z, axis=1)                         # [C, K d], branch k at columns [k d, (k+1) d)
    Wf = np.asarray(Wf, dtype=np.float64)
    E = Zcat @ Wf
    if bf is not None:
        E = E + np.asarray(bf, dtype=np.float64)[None, :]
    return E, dict(outs=outs, caches=caches, rows=rows, Zcat=Zcat)


def mot_backward(dE, branches: List[Branch], n_cand: int, Wf, bf, cache=None):
    """Exact gradient of mot_forward for the loss sum(dE * E).

    Returns (dxs, branch_grads, dWf, dbf): dxs[k] = d loss / d x_k, branch_grads[k][i] the
    gradients of branch k's layer i (oracle.layer_backward keys)."""
    if cache is None:
        _, cache = mot_forward(branches, n_cand, Wf, bf)
    dE = np.asarray(dE, dtype=np.float64)
    Wf = np.asarray(Wf, dtype=np.float64)
    dWf = cache["Zcat"].T @ dE
    dbf = dE.sum(axis=0)
    dZcat = dE @ Wf.T
    d = cache["outs"][0].shape[1]
    dxs, grads = [], []
    for k, br in enumerate(branches):
        dout = np.zeros_like(cache["outs"][k])
        dout[cache["rows"][k]] = dZcat[:, k * d:(k + 1) * d]  # only candidate rows reach E
        dx, g = branch_backward(dout, br, cache["caches"][k])
        dxs.append(dx)
        grads.append(g)
    return dxs, grads, dWf, dbf
