"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NONE of the method's arithmetic: only random draws, the
bf16 (RNE) rounding of those draws (so both sides see identical values), and
the shape/length recipes of DESIGN.md §4.  Every sequence draws
from its own stream ``(seed, seq_id)`` so its content does not depend on which
rank processes it.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

WINDOW_FULL = 2**31 - 1  # "no window limit" (= UH_WINDOW_FULL in include/uhstu.h)


def round_bf16(a: np.ndarray) -> np.ndarray:
    """Round float32 values to the nearest bf16 (ties to even); returns float32."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


def _rng(*key: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence(list(key))))


# ----------------------------------------------------------------------------
# configs (BASELINE.json "configs")
# ----------------------------------------------------------------------------
@dataclass
class Config:
    name: str
    lengths: List[int]
    H: int
    dh: int
    K1: int                  # WINDOW_FULL = causal
    K2: int
    N: float                 # silu(.)/N normaliser (reading R5: configured max length)
    seed: int
    dtype: str = "bf16"
    rab: bool = True
    alpha: float = 1.0
    n_layers: int = 1
    pos_len: int = 0         # P (0 -> N, the configured max length: every offset of the sequence has its own entry, R7)
    ts_len: int = 32         # NB

    @property
    def d(self) -> int:
        return self.H * self.dh

    @property
    def T(self) -> int:
        return int(sum(self.lengths))

    @property
    def P(self) -> int:
        return self.pos_len if self.pos_len else max(1, int(self.N))

    def offsets(self) -> np.ndarray:
        o = np.zeros(len(self.lengths) + 1, dtype=np.int32)
        o[1:] = np.cumsum(self.lengths)
        return o


def lengths_uniform(seed: int, B: int, lo: int, hi: int) -> List[int]:
    return [int(x) for x in _rng(seed, 0xA11).integers(lo, hi + 1, size=B)]


def lengths_loguniform_until(seed: int, lo: int, hi: int, token_budget: int) -> List[int]:
    """Draw log-uniform lengths on [lo, hi] until the budget is met; the last one
    is clipped so the batch holds exactly ``token_budget`` tokens (cfg4)."""
    r = _rng(seed, 0xA12)
    out, tot = [], 0
    while tot < token_budget:
        L = int(np.exp(r.uniform(np.log(lo), np.log(hi))))
        L = min(L, token_budget - tot)
        out.append(L)
        tot += L
    return out


def config(name: str, world: int = 1) -> Config:
    if name == "tiny":
        return Config("tiny", [17, 40, 64], H=2, dh=32, K1=16, K2=2, N=64, seed=0, dtype="f32")
    if name == "tiny128":
        return Config("tiny128", [17, 40, 64], H=2, dh=128, K1=16, K2=2, N=64, seed=0)
    if name == "cfg2":
        return Config("cfg2", lengths_uniform(2, 32, 1024, 4096), H=4, dh=128,
                      K1=WINDOW_FULL, K2=0, N=4096, seed=2)
    if name == "cfg3":
        return Config("cfg3", [16384] * 16 * world, H=4, dh=128, K1=1024, K2=128, N=16384, seed=3)
    if name == "cfg4":
        return Config("cfg4", lengths_loguniform_until(4, 512, 16384, world * 262144), H=4, dh=128,
                      K1=1024, K2=128, N=16384, seed=4, n_layers=18)
    raise KeyError(name)


# ----------------------------------------------------------------------------
# draws
# ----------------------------------------------------------------------------
def timestamps(seed: int, lengths, ids=None) -> np.ndarray:
    """Per sequence: t0 ~ U[1.6e9, 1.7e9] s, gaps floor(exp(U(0, ln 86400))) s.
    ``ids`` are the global sequence ids (default 0..B-1) that key each stream."""
    out = []
    ids = range(len(lengths)) if ids is None else ids
    for i, L in zip(ids, lengths):
        r = _rng(seed, i, 0x7)
        t0 = int(r.integers(1_600_000_000, 1_700_000_000))
        gaps = np.floor(np.exp(r.uniform(0.0, np.log(86400.0), size=max(L - 1, 0)))).astype(np.int64)
        out.append(t0 + np.concatenate([[0], np.cumsum(gaps)]).astype(np.int64)[:L])
    return np.concatenate(out) if out else np.zeros(0, np.int64)


def rows_normal(seed: int, lengths, width: int, std: float, tag: int, ids=None) -> np.ndarray:
    """[T, width] float32 N(0, std^2) rounded to bf16, drawn per sequence (stream (seed, id, tag))."""
    blocks = []
    ids = range(len(lengths)) if ids is None else ids
    for i, L in zip(ids, lengths):
        r = _rng(seed, i, tag)
        blocks.append(r.standard_normal((L, width), dtype=np.float32) * np.float32(std))
    a = np.concatenate(blocks, axis=0) if blocks else np.zeros((0, width), np.float32)
    return round_bf16(a)


def attn_inputs(cfg: Config, seed: Optional[int] = None, ids=None, lengths=None):
    """Q, K ~ N(0, sqrt(4/dh)) elementwise (scores ~ N(0, 2^2)), V ~ N(0,1); bf16-exact."""
    s = cfg.seed if seed is None else seed
    lengths = cfg.lengths if lengths is None else lengths
    sd = (4.0 / cfg.dh) ** 0.25
    q = rows_normal(s, lengths, cfg.d, sd, 0x51, ids)
    k = rows_normal(s, lengths, cfg.d, sd, 0x52, ids)
    v = rows_normal(s, lengths, cfg.d, 1.0, 0x53, ids)
    dA = rows_normal(s, lengths, cfg.d, 1.0, 0x54, ids)
    return q, k, v, dA


def rab_tables(cfg: Config, seed: Optional[int] = None):
    """pos_w ~ N(0, 0.5^2) [P], ts_w ~ N(0, 0.5^2) [NB], float32 (kept fp32 on both sides)."""
    s = cfg.seed if seed is None else seed
    r = _rng(s, 0xB1A5)
    pos = (r.standard_normal(cfg.P) * 0.5).astype(np.float32)
    ts = (r.standard_normal(cfg.ts_len) * 0.5).astype(np.float32)
    return pos, ts


def layer_params(d: int, seed: int, layer: int = 0, biases: bool = True):
    """W1, W2 ~ N(0, 1/d) (bf16-exact); LN gains 1 + 0.1 N, biases 0.1 N (fp32)."""
    r = _rng(seed, 0x1A7E5, layer)
    f = np.float32
    p = dict(
        ln1_w=(1.0 + 0.1 * r.standard_normal(d)).astype(f),
        ln1_b=(0.1 * r.standard_normal(d)).astype(f),
        w1=round_bf16(r.standard_normal((d, 4 * d)).astype(f) / np.sqrt(d)),
        ln2_w=(1.0 + 0.1 * r.standard_normal(d)).astype(f),
        ln2_b=(0.1 * r.standard_normal(d)).astype(f),
        w2=round_bf16(r.standard_normal((d, d)).astype(f) / np.sqrt(d)),
    )
    if biases:
        p["b1"] = (0.1 * r.standard_normal(4 * d)).astype(f)
        p["b2"] = (0.1 * r.standard_normal(d)).astype(f)
    return p


def layer_inputs(cfg: Config, seed: Optional[int] = None, ids=None, lengths=None):
    """x ~ N(0,1) and dOut ~ N(0,1), [T, d], bf16-exact (optionally a subset of sequences)."""
    s = cfg.seed if seed is None else seed
    lengths = cfg.lengths if lengths is None else lengths
    x = rows_normal(s, lengths, cfg.d, 1.0, 0x61, ids)
    dout = rows_normal(s, lengths, cfg.d, 1.0, 0x62, ids)
    return x, dout


def mot_params(d: int, n_branches: int, seed: int):
    """NEXT-4 fusion projection: W_f [K d, d] ~ N(0, 1/(K d)) (bf16-exact), b_f 0.1 N [d] (fp32)."""
    r = _rng(seed, 0x307, n_branches)
    f = np.float32
    w = round_bf16(r.standard_normal((n_branches * d, d)).astype(f) / np.sqrt(n_branches * d))
    return w, (0.1 * r.standard_normal(d)).astype(f)


def mot_lengths(seed: int, B: int, lo: int, hi: int, branch: int) -> List[int]:
    """Per-branch sequence lengths U[lo, hi] for the same B users (branch keys the stream)."""
    r = _rng(seed, 0x3071, branch)
    return [int(v) for v in r.integers(lo, hi + 1, size=B)]
