"""Pins for the LBSL oracle (NEXT-3; Algorithm 1; §4.1), CPU only.

Each pin checks the oracle against something other than itself: SplitMix64's published
output, closed forms (the proxy load is an expectation; the selection-sampling subset
law is uniform over C(n, tau)), brute-force permutation probabilities from the
sequential definition of weighted sampling without replacement, the greedy-fill
bound of Alg. 1 lines 12-16, and the paper's two claims about LBSL: it matches SL's
average load when recalibrated every batch and it lowers the max/min rank-load
ratio."""
import itertools
import math

import numpy as np
import pytest

import lbsl as L


def test_splitmix64_published_vector():
    # SplitMix64 from state 0: the reference outputs of Vigna's splitmix64.c
    assert L.splitmix64_stream(0, 3) == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]


def test_u01_open_interval_and_uniform():
    r = np.array([L.ctr_u01(7, 1, 2, 0, i) for i in range(20000)])
    assert r.min() > 0.0 and r.max() < 1.0
    # mean 1/2 and variance 1/12 within 5 standard errors
    assert abs(r.mean() - 0.5) < 5 * math.sqrt(1 / 12 / len(r))
    assert abs(r.var() - 1 / 12) < 0.003
    # counters are independent: distinct (rank, step, stream) give distinct draws
    assert len({L.ctr_u64(7, a, b, c, 0) for a in range(4) for b in range(4) for c in range(3)}) == 48


def test_rank_load_and_balance():
    assert L.rank_load([2, 2], 2.0) == 8.0
    assert L.rank_load([], 1.5) == 0.0
    assert abs(L.rank_load([3, 5, 7], 1.5) - (3 ** 1.5 + 5 ** 1.5 + 7 ** 1.5)) < 1e-12
    assert L.balance_ratio([5, 5, 5]) == 1.0 and L.balance_ratio([2, 4]) == 2.0
    with pytest.raises(ValueError):
        L.balance_ratio([1.0, 0.0])


def test_standard_sl_truncation_rate_and_proxy_is_expectation():
    """HSTU's SL: P(truncate) = 1 - l_SL^2 / n^2 for n > l_SL (R21); the proxy load is
    E[len^gamma] — a Monte Carlo mean over independent steps converges to it."""
    ell, gamma = 1000, 1.7
    lengths = [500, 1000, 1500, 3000, 8000]
    trials = 4000
    trunc = np.zeros(len(lengths))
    load = 0.0
    for t in range(trials):
        for u, n in enumerate(lengths):
            d = L.standard_sl_decide(n, ell, L.ctr_u01(3, 0, t, L.STREAM_SL, u))
            trunc[u] += d == L.TRUNCATED
            load += float(min(n, ell) if d == L.TRUNCATED else n) ** gamma
    for u, n in enumerate(lengths):
        want = max(0.0, 1 - ell * ell / (n * n))
        assert abs(trunc[u] / trials - want) < 5 * math.sqrt(want * (1 - want) / trials) + 1e-12
    proxy = L.standard_sl_loads(lengths, ell, gamma)
    assert abs(load / trials - proxy) / proxy < 0.03
    # closed form for one user with n = 2 l_SL: q = 1/4
    assert abs(L.standard_sl_loads([2000], 1000, 2.0) - (0.25 * 2000 ** 2 + 0.75 * 1000 ** 2)) < 1e-6


def test_paper_train_length_3072_to_1110():
    """Appendix table: SL maps a 3072-token UIH to 1110 on average. Under R21
    E[len] = q n + (1 - q) l_SL with q = (l_SL/n)^2; solving for l_SL gives ~690, and the
    oracle's sampled mean at that l_SL is 1110 within 1%."""
    n = 3072
    ell = next(l for l in range(1, n) if (l * l / n ** 2) * n + (1 - l * l / n ** 2) * l >= 1110)
    mean = np.mean([min(n, ell) if L.standard_sl_decide(n, ell, L.ctr_u01(11, 0, t, 0, 0)) == L.TRUNCATED
                    else n for t in range(20000)])
    assert abs(mean - 1110) / 1110 < 0.01


def test_sl_subset_increasing_and_uniform():
    n, tau = 10, 4
    counts = {}
    draws = 30000
    for t in range(draws):
        idx = L.sl_subset(n, tau, 5, 0, t, 3)
        assert len(idx) == tau and all(a < b for a, b in zip(idx, idx[1:]))
        counts[tuple(idx)] = counts.get(tuple(idx), 0) + 1
    k = math.comb(n, tau)
    assert len(counts) == k
    exp = draws / k
    chi2 = sum((c - exp) ** 2 / exp for c in counts.values())
    assert chi2 < 209 + 5 * math.sqrt(2 * 209)        # dof = 209
    assert L.sl_subset(5, 5, 1, 0, 0, 0) == [0, 1, 2, 3, 4] and L.sl_subset(5, 0, 1, 0, 0, 0) == []


def test_weighted_permutation_law_matches_sequential_definition():
    """Exponential keys (R24) against brute-force permutation probabilities."""
    p = [1.0, 0.5, 0.25, 0.1]
    perms = list(itertools.permutations(range(4)))
    exact = {pm: L.permutation_prob(p, pm) for pm in perms}
    assert abs(sum(exact.values()) - 1) < 1e-12
    draws = 40000
    cnt = {pm: 0 for pm in perms}
    for t in range(draws):
        cnt[tuple(L.weighted_permutation(p, 9, 0, t))] += 1
    chi2 = sum((cnt[pm] - draws * exact[pm]) ** 2 / (draws * exact[pm]) for pm in perms)
    assert chi2 < 23 + 5 * math.sqrt(46)              # dof = 23
    # equal weights: uniform; a zero-probability-free single element is trivial
    assert L.weighted_permutation([1.0], 1, 0, 0) == [0]


def _pareto_batches(rng, R, b, lo=64, cap=16384, shape=1.5):
    return [[int(min(cap, lo * (1 + rng.pareto(shape)))) for _ in range(b)] for _ in range(R)]


def test_greedy_fill_bound_and_maximality():
    """Alg. 1 lines 12-16: the kept-whole increment s never exceeds the budget, and every
    user left out would have pushed s over it when its turn came."""
    rng = np.random.default_rng(0)
    P = L.LbslParams(R=1, T_warm=1, T_recal=1, gamma=1.7, ell_sl=512, b=32)
    for t in range(50):
        B = _pareto_batches(rng, 1, 32)[0]
        ell_bar = float(rng.uniform(0.8, 3.0)) * 32 * 512.0 ** 1.7
        dec, new = L.rank_select(B, P, ell_bar, True, 4, 0, t)
        budget = ell_bar - sum(min(n, 512) ** 1.7 for n in B)
        U = [u for u in range(32) if dec[u] == L.UNSAMPLED]
        s = sum(B[u] ** 1.7 - min(B[u], 512) ** 1.7 for u in U)
        assert not U or s <= budget + 1e-6 * abs(budget)
        assert all(new[u] == B[u] for u in U)
        assert all(new[u] <= B[u] for u in range(32))
        # realized load = all-truncated baseline + s: capped by l_bar unless the baseline alone exceeds it
        base = sum(min(n, 512) ** 1.7 for n in B)
        realized = L.rank_load(new, 1.7)
        assert abs(realized - (base + s)) <= 1e-9 * realized
        assert realized <= max(ell_bar, base) * (1 + 1e-12)
        # walking pi again: every user outside U would have overrun the budget at its turn
        pi = L.weighted_permutation([L.sl_keep_prob(n, 512) for n in B], 4, 0, t)
        run = 0.0
        for u in pi:
            inc = B[u] ** 1.7 - min(B[u], 512) ** 1.7
            if u in U:
                run += inc
            else:
                assert run + inc > budget


def test_identity_when_l_sl_covers_every_length():
    P = L.LbslParams(R=2, T_warm=2, T_recal=2, gamma=1.5, ell_sl=20000, b=8)
    st = L.LbslState(P)
    rng = np.random.default_rng(1)
    for _ in range(6):
        B = _pareto_batches(rng, 2, 8)
        _, new = L.lbsl_step(st, B, 3)
        assert new == B


def test_target_after_warmup_is_mean_proxy_load():
    """Alg. 1 line 23: l_bar = (1 / (R T_warm)) sum_r l_r after warm-up."""
    P = L.LbslParams(R=3, T_warm=4, T_recal=2, gamma=1.6, ell_sl=300, b=6)
    st = L.LbslState(P)
    rng = np.random.default_rng(2)
    tot = 0.0
    for t in range(4):
        B = _pareto_batches(rng, 3, 6)
        tot += sum(L.standard_sl_loads(b, 300, 1.6) for b in B)
        L.lbsl_step(st, B, 8)
    assert abs(st.ell_bar - tot / 12) <= 1e-12 * tot and st.ell_r == [0.0] * 3


def test_matches_sl_average_load_when_recalibrated_every_batch():
    """recalibrated every batch, LBSL matches standard SL's average load (the
    target is last batch's mean proxy load, so it is checked over R = 8 ranks)."""
    P = L.LbslParams(R=8, T_warm=5, T_recal=1, gamma=1.7, ell_sl=512, b=32)
    st = L.LbslState(P)
    rng = np.random.default_rng(3)
    lb, sl = [], []
    for t in range(1, 81):
        B = _pareto_batches(rng, 8, 32, lo=256)
        sl_t = L.standard_sl_step(B, P, 21, t)
        _, new = L.lbsl_step(st, B, 21)
        if t > P.T_warm:
            sl += [L.rank_load(x, 1.7) for x in sl_t]
            lb += [L.rank_load(x, 1.7) for x in new]
    assert abs(np.mean(lb) - np.mean(sl)) / np.mean(sl) < 0.05


def test_lbsl_lowers_rank_load_imbalance():
    """LBSL reduces the max/min rank-load ratio against SL on the same stream."""
    R, b = 8, 32
    P = L.LbslParams(R=R, T_warm=20, T_recal=10, gamma=1.7, ell_sl=512, b=b)
    st = L.LbslState(P)
    rng = np.random.default_rng(4)
    r_lb, r_sl = [], []
    for t in range(1, 121):
        B = _pareto_batches(rng, R, b, lo=256)
        sl = L.standard_sl_step(B, P, 5, t)
        _, new = L.lbsl_step(st, B, 5)
        if t > 40:
            r_sl.append(L.balance_ratio([L.rank_load(x, 1.7) for x in sl]))
            r_lb.append(L.balance_ratio([L.rank_load(x, 1.7) for x in new]))
    assert np.mean(r_lb) < 0.8 * np.mean(r_sl) and np.mean(r_lb) < 1.2
