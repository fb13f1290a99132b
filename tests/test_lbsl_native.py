"""NEXT-3 LBSL: the native library (include/uhstu_lbsl.h) against the oracle
(oracle/lbsl.py, Alg. 1), bit for bit — both implement the same counter-based
generator, so decisions, realized lengths, subsets and row lists must be identical and
the proxy loads equal in fp64.  Host code only: runs without a GPU.  The device gather is
checked in test_gpu_lbsl.py; the world-size-2 target all-reduce here over gloo."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import lbsl as OL
from paper_2602_16986_b200 import lbsl as NL
from paper_2602_16986_b200 import uhstu as U


def _pareto(rng, b, lo=64, cap=16384, shape=1.5):
    return [int(min(cap, lo * (1 + rng.pareto(shape)))) for _ in range(b)]


@pytest.mark.parametrize("steady", [False, True])
def test_select_matches_oracle_bit_exact(steady):
    rng = np.random.default_rng(10 + steady)
    for trial in range(300):
        b = int(rng.integers(0, 40))
        B = _pareto(rng, b, lo=int(rng.choice([1, 64, 256])))
        if trial % 7 == 0 and b:
            B[0] = 0                                            # empty history
        ell = int(rng.choice([1, 100, 512, 700]))
        gamma = float(rng.uniform(1.05, 1.95))
        ell_bar = float(rng.uniform(0.0, 3.0)) * max(b, 1) * ell ** gamma
        seed, rank, t = int(rng.integers(0, 2 ** 63)), int(rng.integers(0, 512)), int(rng.integers(1, 10 ** 6))
        P = OL.LbslParams(R=1, T_warm=1, T_recal=1, gamma=gamma, ell_sl=ell, b=b)
        od, on = OL.rank_select(B, P, ell_bar, steady, seed, rank, t)
        nd, nn, proxy = U.lbsl_select(B, ell, gamma, ell_bar, steady, seed, rank, t)
        assert list(nd) == od and list(nn) == on
        assert proxy == OL.standard_sl_loads(B, ell, gamma)


def test_subset_and_rows_match_oracle():
    rng = np.random.default_rng(3)
    for trial in range(60):
        n = int(rng.integers(0, 300))
        tau = int(rng.integers(0, n + 1))
        seed, rank, t, u = int(rng.integers(0, 2 ** 63)), int(rng.integers(0, 8)), int(rng.integers(1, 999)), \
            int(rng.integers(0, 64))
        assert list(U.lbsl_subset(n, tau, seed, rank, t, u)) == OL.sl_subset(n, tau, seed, rank, t, u)
    # whole-step row list: users in order, kept positions ascending
    B = _pareto(rng, 32, lo=256)
    off = np.concatenate([[0], np.cumsum(B)]).astype(np.int32)
    P = OL.LbslParams(R=1, T_warm=1, T_recal=1, gamma=1.7, ell_sl=512, b=32)
    dec, new = OL.rank_select(B, P, 32 * 700 ** 1.7, True, 99, 2, 17)
    want = []
    for u in range(32):
        pos = OL.sl_subset(B[u], new[u], 99, 2, 17, u) if dec[u] == OL.TRUNCATED else range(B[u])
        want += [off[u] + j for j in pos]
    rows, new_off = U.lbsl_rows(off, dec, new, 99, 2, 17)
    assert list(rows) == want and list(np.diff(new_off)) == new and new_off[0] == 0


def test_argument_errors():
    with pytest.raises(U.UhError):
        U.lbsl_select([3, -1], 4, 1.5, 0.0, False, 0, 0, 1)
    with pytest.raises(U.UhError):
        U.lbsl_select([3], 0, 1.5, 0.0, False, 0, 0, 1)
    with pytest.raises(U.UhError):
        U.lbsl_subset(3, 4, 0, 0, 1, 0)
    with pytest.raises(U.UhError):
        U.lbsl_rows([0, 5], [0], [6], 0, 0, 1)                 # truncated longer than the history
    d, n, p = U.lbsl_select([], 4, 1.5, 0.0, True, 0, 0, 1)
    assert len(d) == 0 and p == 0.0


def test_runtime_single_rank_matches_oracle_steps():
    """The LBSL runtime (state machine + native selection) against oracle lbsl_step, R = 1."""
    cfg = NL.LbslConfig(T_warm=4, T_recal=3, gamma=1.6, ell_sl=300, seed=5)
    rt = NL.LBSL(cfg)
    st = OL.LbslState(OL.LbslParams(R=1, T_warm=4, T_recal=3, gamma=1.6, ell_sl=300, b=16))
    rng = np.random.default_rng(8)
    for t in range(20):
        B = _pareto(rng, 16, lo=128)
        od, on = OL.lbsl_step(st, [B], 5)
        nd, nn = rt.select(B)
        assert list(nd) == od[0] and list(nn) == on[0]
        assert rt.ell_bar == st.ell_bar


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rt = NL.LBSL(NL.LbslConfig(T_warm=3, T_recal=2, gamma=1.7, ell_sl=400, seed=13), rank=rank, world=world)
        rng = np.random.default_rng(100)
        out = []
        for t in range(10):
            batches = [_pareto(rng, 12, lo=200) for _ in range(world)]
            d, n = rt.select(batches[rank])
            out.append((list(n), rt.ell_bar))
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_two_ranks_gloo_match_oracle_world():
    """world_size 2 over gloo: each rank's realized lengths and the all-reduced target equal
    the oracle's in-process R = 2 simulation of Algorithm 1."""
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=180) for _ in ps)
    for p in ps:
        p.join(60)
        assert p.exitcode == 0
    st = OL.LbslState(OL.LbslParams(R=2, T_warm=3, T_recal=2, gamma=1.7, ell_sl=400, b=12))
    rng = np.random.default_rng(100)
    for t in range(10):
        batches = [_pareto(rng, 12, lo=200) for _ in range(world)]
        _, on = OL.lbsl_step(st, batches, 13)
        for r in range(world):
            n, ell_bar = res[r][t]
            assert n == on[r]
            assert abs(ell_bar - st.ell_bar) <= 1e-12 * max(1.0, st.ell_bar)
