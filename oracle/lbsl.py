"""ORACLE — test infrastructure only (NEXT-3: Load-Balanced Stochastic Length).

Plain Python implementation of LBSL, Algorithm 1 (App. C) and
§4.1, in the algorithm's order and notation.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s baseline legs may import it; it shares
no code with the native implementation (``csrc/lbsl.cu``) and neither imports the
other.  Both sides implement the same counter-based generator (``ctr_u01`` below,
DESIGN.md R24), so the random draws are identical and the decisions comparable bit
for bit.

Readings:
* R21 StandardSL (after HSTU's SL): a user with n_u > l_SL is truncated to
  l_SL tokens with probability 1 - (l_SL / n_u)^2 and kept whole otherwise
  (l_SL = L^{alpha/2}, so (l_SL/n_u)^2 = L^alpha / n_u^2); n_u <= l_SL is never touched.
  The truncated sequence is a uniformly random order-preserving subset of l_SL of the
  n_u positions (selection sampling, Knuth's Algorithm S).
* R22 SLWeight(n_u; alpha) = the probability StandardSL leaves u unsampled,
  min(1, (l_SL / n_u)^2) — "SL's bias toward leaving shorter sequences unsampled"
  (P:113).  StandardSL_Loads (Alg. 1 line 5, "pre-truncation proxy") = the expected
  StandardSL load sum_u E[len_u^gamma], computed from the raw lengths before any draw.
* R23 Recalibration (Alg. 1 lines 22-27) runs only after warm-up (t > T_warm), and
  divides by the number of steps accumulated since the last reset (= T_recal when
  T_warm is a multiple of T_recal); the literal text would recalibrate inside the
  warm-up and divide by T_warm a sum that was reset at the last multiple of T_recal.
* R25 The greedy fill's baseline (Alg. 1 line 13): b * l_SL^gamma is the load of the
  batch with every example truncated to l_SL, which holds when every n_u >= l_SL (the
  paper's regime).  Examples shorter than l_SL are never truncated, so the baseline
  is read as sum_u min(n_u, l_SL)^gamma and the increment as n_u^gamma -
  min(n_u, l_SL)^gamma — identical to the printed text when all n_u >= l_SL; the
  literal text makes the budget negative for batches of short users and LBSL
  collapse to plain SL.  Sums run in index order.
* R26 "For each u not in U_r, apply the same sampling rule as StandardSL" (Alg. 1
  line 18) is read as SL's *sampling* (truncation to l_SL by R21's subset), not its
  random keep-or-truncate choice: U_r is what replaces that choice.  Then each rank's
  realized load is sum_u min(n_u, l_SL)^gamma + s <= l_bar, "so each rank's realized
  load matches l as closely as possible"; with SL's random choice kept the
  heavy ranks would overshoot l_bar and the load would not be controlled.
* R24 Weighted permutation without replacement (Alg. 1 line 11) by exponential keys
  (Efraimidis-Spirakis): key_u = log(r_u) / p_u, larger first, ties by index.  Its
  law is pinned against the sequential definition by brute force in the tests.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Sequence, Tuple

M64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15

STREAM_SL = 0      # StandardSL truncate / keep decision of user u
STREAM_PERM = 1    # weighted-permutation key of user u
STREAM_SUBSET = 2  # selection-sampling draws for the positions of user u

TRUNCATED, KEPT_BY_SL, UNSAMPLED = 0, 1, 2


def mix64(z: int) -> int:
    """SplitMix64 finaliser (Steele, Lea, Flood 2014)."""
    z &= M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def splitmix64_stream(state: int, n: int) -> List[int]:
    """The first n outputs of SplitMix64 from ``state`` (pinned to its published vector)."""
    out = []
    for _ in range(n):
        state = (state + GOLDEN) & M64
        out.append(mix64(state))
    return out


def ctr_u64(seed: int, rank: int, step: int, stream: int, idx: int) -> int:
    """Counter-based draw: the SplitMix64 finaliser chained over (rank, step, stream, idx)."""
    x = seed & M64
    for c in (rank, step, stream, idx):
        x = mix64((x + GOLDEN + (c & M64)) & M64)
    return x


def ctr_u01(seed: int, rank: int, step: int, stream: int, idx: int) -> float:
    """Uniform in the open interval (0, 1): the top 53 bits, centred in their cell."""
    return ((ctr_u64(seed, rank, step, stream, idx) >> 11) + 0.5) * 2.0 ** -53


# ------------------------------------------------------------------ §4.1 definitions
def rank_load(lengths: Sequence[int], gamma: float) -> float:
    """Load of a rank in a batch: sum_u n_u^gamma."""
    s = 0.0
    for n in lengths:
        s += float(n) ** gamma
    return s


def balance_ratio(loads: Sequence[float]) -> float:
    """Max / min rank load within a world."""
    if min(loads) <= 0:
        raise ValueError("balance ratio needs positive loads")
    return max(loads) / min(loads)


def sl_keep_prob(n: int, ell_sl: int) -> float:
    """R21/R22: probability StandardSL leaves u unsampled; also SLWeight(n_u; alpha)."""
    if n <= ell_sl:
        return 1.0
    return (float(ell_sl) * float(ell_sl)) / (float(n) * float(n))


def standard_sl_loads(lengths: Sequence[int], ell_sl: int, gamma: float) -> float:
    """R22: StandardSL_Loads(B_r; alpha; gamma) = sum_u E[len_u^gamma] under StandardSL."""
    s = 0.0
    for n in lengths:
        if n <= ell_sl:
            s += float(n) ** gamma
        else:
            q = sl_keep_prob(n, ell_sl)
            s += q * float(n) ** gamma + (1.0 - q) * float(ell_sl) ** gamma
    return s


def standard_sl_decide(n: int, ell_sl: int, r: float) -> int:
    """R21 for one user with its uniform draw r: truncate iff n > l_SL and r >= q_u."""
    if n > ell_sl and r >= sl_keep_prob(n, ell_sl):
        return TRUNCATED
    return KEPT_BY_SL


def sl_subset(n: int, tau: int, seed: int, rank: int, step: int, u: int) -> List[int]:
    """R21: a uniformly random order-preserving subset of tau of range(n), by Knuth's
    selection sampling: position j is taken with probability (needed) / (remaining)."""
    idx = []
    for j in range(n):
        r = ctr_u01(seed, rank, step, STREAM_SUBSET, (u << 32) | j)
        if float(n - j) * r < float(tau - len(idx)):
            idx.append(j)
    return idx


def weighted_permutation(p: Sequence[float], seed: int, rank: int, step: int) -> List[int]:
    """R24: Alg. 1 line 11, weighted random permutation without replacement."""
    keys = [math.log(ctr_u01(seed, rank, step, STREAM_PERM, u)) / p[u] for u in range(len(p))]
    return sorted(range(len(p)), key=lambda u: (-keys[u], u))


def permutation_prob(p: Sequence[float], perm: Sequence[int]) -> float:
    """The sequential definition of weighted sampling without replacement: each next
    element is drawn with probability proportional to its weight among those left."""
    left = list(range(len(p)))
    prob = 1.0
    for u in perm:
        prob *= p[u] / sum(p[v] for v in left)
        left.remove(u)
    return prob


# ------------------------------------------------------------------ Algorithm 1
@dataclass
class LbslParams:
    R: int
    T_warm: int
    T_recal: int
    gamma: float
    ell_sl: int
    b: int


@dataclass
class LbslState:
    params: LbslParams
    ell_bar: float = 0.0                                  # target load (line 1)
    ell_r: List[float] = field(default_factory=list)      # per-rank accumulators (line 1)
    t: int = 0                                            # last finished step
    since_reset: int = 0                                  # steps in ell_r (R23)

    def __post_init__(self):
        if not self.ell_r:
            self.ell_r = [0.0] * self.params.R


def rank_select(lengths: Sequence[int], P: LbslParams, ell_bar: float, steady: bool,
                seed: int, rank: int, t: int) -> Tuple[List[int], List[int]]:
    """Alg. 1 lines 4-20 for one rank: the per-example decision and realized length."""
    b = len(lengths)
    decision = [KEPT_BY_SL] * b
    if steady:
        U = set()                                           # line 9
        s = 0.0
        p = [sl_keep_prob(n, P.ell_sl) for n in lengths]   # line 10
        pi = weighted_permutation(p, seed, rank, t)         # line 11
        base = [float(min(n, P.ell_sl)) ** P.gamma for n in lengths]   # R25
        budget = ell_bar - sum(base)
        for u in pi:                                        # lines 12-16
            inc = float(lengths[u]) ** P.gamma - base[u]
            if s + inc <= budget:
                U.add(u)
                s = s + inc
        for u in range(b):                                  # lines 17-18
            if u in U:
                decision[u] = UNSAMPLED
            else:                                           # R26
                decision[u] = TRUNCATED if lengths[u] > P.ell_sl else KEPT_BY_SL
    else:                                                   # line 7
        for u in range(b):
            decision[u] = standard_sl_decide(lengths[u], P.ell_sl, ctr_u01(seed, rank, t, STREAM_SL, u))
    new_len = [min(n, P.ell_sl) if dcs == TRUNCATED else n for n, dcs in zip(lengths, decision)]
    return decision, new_len


def lbsl_step(state: LbslState, batches: Sequence[Sequence[int]], seed: int):
    """One training step of Algorithm 1 over all R ranks (simulated in-process; the
    all-reduce of lines 22/25 is the in-process sum).  Returns (decisions, new_lens)."""
    P = state.params
    t = state.t + 1                                         # line 2
    steady = t > P.T_warm
    decisions, new_lens = [], []
    for r in range(P.R):                                    # line 3
        B_r = batches[r]                                    # line 4
        state.ell_r[r] += standard_sl_loads(B_r, P.ell_sl, P.gamma)   # line 5
        d, nl = rank_select(B_r, P, state.ell_bar, steady, seed, r, t)
        decisions.append(d)
        new_lens.append(nl)
    state.since_reset += 1
    if t == P.T_warm or (t > P.T_warm and t % P.T_recal == 0):       # lines 22-27, R23
        state.ell_bar = sum(state.ell_r) / (P.R * state.since_reset)
        state.ell_r = [0.0] * P.R
        state.since_reset = 0
    state.t = t
    return decisions, new_lens


def standard_sl_step(batches: Sequence[Sequence[int]], P: LbslParams, seed: int, t: int):
    """Plain StandardSL on every rank (the paper's baseline), same draws."""
    return [rank_select(B_r, P, 0.0, False, seed, r, t)[1] for r, B_r in enumerate(batches)]
