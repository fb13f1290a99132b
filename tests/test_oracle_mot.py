"""Pins for the MoT oracle (NEXT-4; readings R28-R30), CPU only.

Each pin checks oracle/mot.py against something other than itself: a hand-written row map
(R29's candidate positions), brute-force sums for the projection, selector projections that
must return one branch's candidate outputs unchanged (the concatenation order), an averaging
projection over two identical branches that must equal one branch (the paper's "fuses the
learned user embeddings" degenerates to the single transducer), user independence (a change
in one user's history leaves every other user's embeddings bit-identical), and central
finite differences for every gradient the backward returns."""
import numpy as np
import pytest

import mot as M
import oracle as O
from paper_2602_16986_b200 import synth


def _branch(seed, lengths, n_layers, H=2, dh=3, K1=2, K2=1, rab=True):
    d = H * dh
    off = np.zeros(len(lengths) + 1, np.int32)
    off[1:] = np.cumsum(lengths)
    r = np.random.default_rng(seed)
    layers = []
    for i in range(n_layers):
        p = synth.layer_params(d, seed, layer=i)
        prm = O.LayerParams(**{k: np.asarray(v, np.float64) for k, v in p.items()})
        spec = O.AttnSpec(K1=K1, K2=K2, alpha=0.8, N=9.0)
        if rab:
            spec.pos_w = r.standard_normal(8) * 0.5
            spec.ts_w = r.standard_normal(6) * 0.5
            spec.timestamps = synth.timestamps(seed, lengths)
        layers.append((prm, H, spec))
    x = r.standard_normal((int(off[-1]), d))
    return M.Branch(x=x, offsets=off, layers=layers)


def _two(n_cand=2):
    a = _branch(1, (5, 7, 3), 2)                        # "C-seq": deeper, longer
    b = _branch(2, (4, 3, 6), 1, K1=O.FULL, K2=0)       # "E-seq": shallower, full causal
    W, bias = synth.mot_params(6, 2, 3)
    return [a, b], n_cand, np.asarray(W, np.float64), np.asarray(bias, np.float64)


def test_candidate_rows_hand_written():
    # offsets [0, 5, 9, 12], two candidates per user: rows 3,4 | 7,8 | 10,11
    assert M.candidate_rows([0, 5, 9, 12], 2).tolist() == [3, 4, 7, 8, 10, 11]
    assert M.candidate_rows([0, 1], 1).tolist() == [0]
    with pytest.raises(ValueError):
        M.candidate_rows([0, 5, 6], 2)              # second user has one row
    with pytest.raises(ValueError):
        M.candidate_rows([0, 5], 0)


def test_projection_brute_force():
    brs, nc, W, bias = _two()
    E, cache = M.mot_forward(brs, nc, W, bias)
    outs = [M.branch_forward(b)[0] for b in brs]
    rows = [M.candidate_rows(b.offsets, nc) for b in brs]
    d = W.shape[1]
    for c in (0, 3, 5):
        for n in (0, 4):
            want = bias[n]
            for k in range(2):
                for i in range(d):
                    want += outs[k][rows[k][c], i] * W[k * d + i, n]
            assert abs(E[c, n] - want) < 1e-12


def test_selector_projections_return_one_branch():
    brs, nc, W, _ = _two()
    d = W.shape[1]
    I, Z = np.eye(d), np.zeros((d, d))
    for k in range(2):
        sel = np.concatenate([I if j == k else Z for j in range(2)], axis=0)
        E, _ = M.mot_forward(brs, nc, sel, None)
        out, _ = M.branch_forward(brs[k])
        assert np.array_equal(E, out[M.candidate_rows(brs[k].offsets, nc)])


def test_identical_branches_average_equals_single_branch():
    a = _branch(4, (6, 5), 2)
    d = 6
    avg = np.concatenate([np.eye(d) / 2, np.eye(d) / 2], axis=0)
    E2, _ = M.mot_forward([a, a], 3, avg, None)
    E1, _ = M.mot_forward([a], 3, np.eye(d), None)
    assert np.max(np.abs(E2 - E1)) < 1e-13


def test_user_independence():
    brs, nc, W, bias = _two()
    E, _ = M.mot_forward(brs, nc, W, bias)
    b2 = M.Branch(x=brs[1].x.copy(), offsets=brs[1].offsets, layers=brs[1].layers)
    b2.x[4, 0] += 1.0                                   # user 1's history in branch 1 (rows 4..6)
    E2, _ = M.mot_forward([brs[0], b2], nc, W, bias)
    assert np.array_equal(E[:nc], E2[:nc]) and np.array_equal(E[2 * nc:], E2[2 * nc:])
    assert np.max(np.abs(E[nc:2 * nc] - E2[nc:2 * nc])) > 1e-6


def test_mismatched_users_rejected():
    a = _branch(1, (5, 7), 1)
    b = _branch(2, (4, 3, 6), 1)
    with pytest.raises(ValueError):
        M.mot_forward([a, b], 2, np.zeros((12, 6)), None)


def _loss(brs, nc, W, bias, dE):
    E, _ = M.mot_forward(brs, nc, W, bias)
    return float(np.sum(E * dE))


def test_backward_finite_differences():
    brs, nc, W, bias = _two()
    r = np.random.default_rng(9)
    E, cache = M.mot_forward(brs, nc, W, bias)
    dE = r.standard_normal(E.shape)
    dxs, grads, dW, db = M.mot_backward(dE, brs, nc, W, bias, cache=cache)
    h = 1e-6

    def fd(f, arr, idx):
        old = arr[idx]
        arr[idx] = old + h
        up = f()
        arr[idx] = old - h
        dn = f()
        arr[idx] = old
        return (up - dn) / (2 * h)

    L = lambda: _loss(brs, nc, W, bias, dE)
    for idx in [(0, 0), (7, 3), (11, 5)]:
        assert abs(fd(L, W, idx) - dW[idx]) < 1e-6 * max(1.0, abs(dW[idx]))
    for idx in [(0,), (4,)]:
        assert abs(fd(L, bias, idx) - db[idx]) < 1e-6 * max(1.0, abs(db[idx]))
    # inputs: candidate rows, history rows of both branches (history reaches E through attention)
    for k, rows in ((0, (0, 4, 9, 14)), (1, (0, 3, 6, 12))):
        for row in rows:
            idx = (row, 2)
            g = fd(L, brs[k].x, idx)
            assert abs(g - dxs[k][idx]) < 1e-6 * max(1.0, abs(g)), (k, row, g, dxs[k][idx])
    # a parameter of each branch's first layer and of branch 0's last layer
    for k, li, name, idx in ((0, 0, "w1", (1, 7)), (0, 1, "w2", (2, 3)), (1, 0, "ln1_w", (4,)),
                             (0, 0, "pos_w", (1,))):
        prm, H, spec = brs[k].layers[li]
        arr = spec.pos_w if name == "pos_w" else getattr(prm, name)
        g = fd(L, arr, idx)
        assert abs(g - grads[k][li][name][idx]) < 1e-6 * max(1.0, abs(g)), (k, li, name, g)


def test_every_row_a_candidate_is_a_plain_projection():
    """n_cand = L for every sequence: the fusion is the row-aligned concatenation of the branch
    outputs times W_f (checked against an explicit matmul of the stacked outputs)."""
    a = _branch(5, (4, 6), 1)
    b = _branch(6, (4, 6), 2, K1=O.FULL, K2=0)
    W, bias = synth.mot_params(6, 2, 8)
    W, bias = np.asarray(W, np.float64), np.asarray(bias, np.float64)
    E, _ = M.mot_forward([a, b], 4, W, bias)          # n_cand = 4 = shortest length; rows 2..5 of user 1
    oa, _ = M.branch_forward(a)
    ob, _ = M.branch_forward(b)
    rows = np.r_[0:4, 6:10]
    want = np.concatenate([oa[rows], ob[rows]], axis=1) @ W + bias
    assert np.max(np.abs(E - want)) < 1e-12
