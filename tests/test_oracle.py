"""Pins for the fp64 oracle (oracle/), run on CPU (-m "not gpu").

Each test pins the oracle to something other than itself: a hand-written golden
fixture, a closed form, a textbook special case, a library routine (torch fp64
autograd / layer_norm), a dense fully-materialised formulation, or central finite
differences.  A dropped term, wrong sign, wrong index or transposed operand in
oracle/attn_oracle.c or oracle/oracle.py fails at least one of them.
"""
import os

import numpy as np
import pytest
import torch

import oracle as O
from paper_2602_16986_b200 import synth

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# ---------------------------------------------------------------------------
# independent dense constructions (matrix ops, not the oracle's predicate)
# ---------------------------------------------------------------------------
def dense_mask(L, K1, K2):
    """Causal lower triangle AND (band of width K1 OR first K2 columns), built with tril/triu."""
    causal = np.tril(np.ones((L, L), bool))
    if K1 < 0:
        return causal
    band = np.triu(np.ones((L, L), bool), k=-K1)
    glob = np.zeros((L, L), bool)
    glob[:, :K2] = True
    return causal & (band | glob)


def dense_attention(offsets, H, dh, q, k, v, K1, K2, alpha, N, pos=None, ts=None, t=None):
    """Fully materialised per-(sequence, head) attention in torch fp64."""
    out = np.zeros((offsets[-1], H * dh))
    for b in range(len(offsets) - 1):
        o0, o1 = offsets[b], offsets[b + 1]
        L = o1 - o0
        if L == 0:
            continue
        M = torch.from_numpy(dense_mask(L, K1, K2))
        bias = torch.zeros(L, L, dtype=torch.float64)
        if pos is not None:
            P = len(pos)
            dist = torch.arange(L)[:, None] - torch.arange(L)[None, :]
            bias += torch.from_numpy(np.asarray(pos, np.float64))[dist.clamp(0, P - 1)]
        if ts is not None:
            tt = torch.from_numpy(np.asarray(t[o0:o1], np.float64))
            delta = (tt[:, None] - tt[None, :]).clamp(min=1.0)
            bk = torch.floor(torch.log2(delta)).long().clamp(0, len(ts) - 1)
            bias += torch.from_numpy(np.asarray(ts, np.float64))[bk]
        for h in range(H):
            sl = slice(h * dh, (h + 1) * dh)
            Q = torch.from_numpy(np.asarray(q[o0:o1, sl], np.float64))
            K = torch.from_numpy(np.asarray(k[o0:o1, sl], np.float64))
            V = torch.from_numpy(np.asarray(v[o0:o1, sl], np.float64))
            S = alpha * Q @ K.T + bias
            P_ = torch.nn.functional.silu(S) / N
            P_ = torch.where(M, P_, torch.zeros_like(P_))
            out[o0:o1, sl] = (P_ @ V).numpy()
    return out


def rel_inf(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def small_case(lengths=(5, 7, 1, 12), H=2, dh=3, seed=11, rab=True):
    r = np.random.default_rng(seed)
    off = np.zeros(len(lengths) + 1, np.int32)
    off[1:] = np.cumsum(lengths)
    T = off[-1]
    q = r.standard_normal((T, H * dh)); k = r.standard_normal((T, H * dh)); v = r.standard_normal((T, H * dh))
    spec = O.AttnSpec(K1=2, K2=1, alpha=0.7, N=9.0)
    if rab:
        spec.pos_w = r.standard_normal(6) * 0.5
        spec.ts_w = r.standard_normal(5) * 0.5
        spec.timestamps = synth.timestamps(seed, lengths)
    return off, q, k, v, spec


# ---------------------------------------------------------------------------
# mask
# ---------------------------------------------------------------------------
def test_mask_golden_L6():
    rows = [l.split() for l in open(os.path.join(GOLDEN, "sla_mask_L6_K1_2_K2_2.txt")) if not l.startswith("#")]
    gold = np.array(rows, dtype=int)
    got = np.array([[O.mask_allows(q, k, 2, 2) for k in range(6)] for q in range(6)], dtype=int)
    assert (got == gold).all()


def closed_form_nnz(L, K1, K2):
    """SURVEY App. A closed form, derived independently of the enumeration."""
    if K1 < 0:
        return L * (L + 1) // 2
    m = min(L, K1 + 1)
    R = L - 1 - K1
    n = m * (m + 1) // 2 + (L - m) * (K1 + 1)
    if R > 0:
        m2 = min(R, K2)
        n += m2 * (m2 + 1) // 2 + (R - m2) * K2
    return n


def test_mask_nnz_closed_form_and_dense():
    for L in range(0, 41):
        for K1 in list(range(0, L + 2)) + [O.FULL]:
            for K2 in range(0, L + 2, 3):
                n = O.mask_nnz(L, K1, K2)
                assert n == closed_form_nnz(L, K1, K2), (L, K1, K2)
                if L <= 24:
                    assert n == int(dense_mask(L, K1, K2).sum())


def test_mask_special_cases():
    assert O.mask_nnz(4, O.FULL, 0) == 10
    assert O.mask_nnz(5, 1, 0) == 9
    for L in (1, 7, 33):
        assert O.mask_nnz(L, 0, 0) == L                      # diagonal only
        assert O.mask_nnz(L, L - 1, 0) == L * (L + 1) // 2   # window covers the triangle
    # the survey's worked numbers: tiny per-head nnz and cfg3 per-sequence nnz
    assert O.mask_nnz(17, 16, 2) + O.mask_nnz(40, 16, 2) + O.mask_nnz(64, 16, 2) == 1787
    assert closed_form_nnz(16384, 1024, 128) == 18226624


def test_mask_linearity():
    # O((K1+K2) L) claim
    K1, K2 = 16, 4
    for L in (256, 1000, 4000):  # L >> K1+K2 so boundary terms are small
        r = O.mask_nnz(2 * L, K1, K2) / O.mask_nnz(L, K1, K2)
        assert 1.9 <= r <= 2.1


# ---------------------------------------------------------------------------
# attention forward (Eq. 3)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("rab", [False, True])
def test_attention_matches_dense(rab):
    off, q, k, v, spec = small_case(rab=rab)
    A, work = O.attention_forward(off, 2, 3, q, k, v, spec, return_work=True)
    D = dense_attention(off, 2, 3, q, k, v, spec.K1, spec.K2, spec.alpha, spec.N,
                        spec.pos_w, spec.ts_w, spec.timestamps)
    assert np.max(np.abs(A - D)) < 1e-12
    L = np.diff(off)
    assert work == 2 * sum(closed_form_nnz(int(l), spec.K1, spec.K2) for l in L)


def test_attention_tiny_config_dense():
    cfg = synth.config("tiny")
    q, k, v, _ = synth.attn_inputs(cfg)
    pos, ts = synth.rab_tables(cfg)
    t = synth.timestamps(cfg.seed, cfg.lengths)
    spec = O.AttnSpec(K1=cfg.K1, K2=cfg.K2, alpha=1.0, N=cfg.N, pos_w=pos, ts_w=ts, timestamps=t)
    A = O.attention_forward(cfg.offsets(), cfg.H, cfg.dh, q, k, v, spec)
    D = dense_attention(cfg.offsets(), cfg.H, cfg.dh, q, k, v, cfg.K1, cfg.K2, 1.0, cfg.N, pos, ts, t)
    assert rel_inf(A, D) < 1e-12


def test_attention_L1_closed_form():
    r = np.random.default_rng(3)
    q, k, v = r.standard_normal((1, 4)), r.standard_normal((1, 4)), r.standard_normal((1, 4))
    pos = np.array([0.3, -1.0]); ts = np.array([0.2, 0.5])
    spec = O.AttnSpec(K1=5, K2=2, alpha=0.5, N=3.0, pos_w=pos, ts_w=ts, timestamps=np.array([100], np.int64))
    A = O.attention_forward(np.array([0, 1]), 1, 4, q, k, v, spec)
    s = 0.5 * float(q[0] @ k[0]) + 0.3 + 0.2
    assert np.allclose(A[0], s / (1 + np.exp(-s)) / 3.0 * v[0], rtol=0, atol=1e-14)


def test_attention_zero_v_and_diagonal_only():
    off, q, k, v, spec = small_case()
    assert np.all(O.attention_forward(off, 2, 3, q, k, 0 * v, spec) == 0.0)
    spec0 = O.AttnSpec(K1=0, K2=0, alpha=1.3, N=2.0)
    A = O.attention_forward(off, 2, 3, q, k, v, spec0)
    for h in range(2):
        sl = slice(3 * h, 3 * h + 3)
        s = 1.3 * np.sum(q[:, sl] * k[:, sl], axis=1)
        exp = (s / (1 + np.exp(-s)) / 2.0)[:, None] * v[:, sl]
        assert np.max(np.abs(A[:, sl] - exp)) < 1e-14


def test_window_geq_L_equals_full_causal():
    # north star invariant: window >= L with zero global tokens == full causal
    off, q, k, v, spec = small_case(rab=True)
    spec_w = O.AttnSpec(K1=100, K2=0, alpha=spec.alpha, N=spec.N, pos_w=spec.pos_w,
                        ts_w=spec.ts_w, timestamps=spec.timestamps)
    spec_c = O.AttnSpec(K1=O.FULL, K2=0, alpha=spec.alpha, N=spec.N, pos_w=spec.pos_w,
                        ts_w=spec.ts_w, timestamps=spec.timestamps)
    a = O.attention_forward(off, 2, 3, q, k, v, spec_w)
    b = O.attention_forward(off, 2, 3, q, k, v, spec_c)
    assert np.array_equal(a, b)
    # and full causal == the dense lower-triangular formulation
    D = dense_attention(off, 2, 3, q, k, v, O.FULL, 0, spec.alpha, spec.N, spec.pos_w, spec.ts_w, spec.timestamps)
    assert np.max(np.abs(b - D)) < 1e-12


def test_jagged_equals_padded():
    off, q, k, v, spec = small_case(rab=False)
    A = O.attention_forward(off, 2, 3, q, k, v, spec)
    # pad every sequence with 3 trailing garbage tokens; real rows must not change
    r = np.random.default_rng(5)
    rows_q, rows_k, rows_v, offp, keep = [], [], [], [0], []
    for b in range(len(off) - 1):
        o0, o1 = off[b], off[b + 1]
        for src, dst in ((q, rows_q), (k, rows_k), (v, rows_v)):
            dst.append(src[o0:o1]); dst.append(r.standard_normal((3, src.shape[1])))
        keep.extend(range(offp[-1], offp[-1] + (o1 - o0)))
        offp.append(offp[-1] + (o1 - o0) + 3)
    Ap = O.attention_forward(np.array(offp), 2, 3, np.concatenate(rows_q), np.concatenate(rows_k),
                             np.concatenate(rows_v), spec)
    assert np.array_equal(Ap[keep], A)


def test_causality_perturbation():
    off, q, k, v, spec = small_case(rab=True)
    A = O.attention_forward(off, 2, 3, q, k, v, spec)
    b = 3  # last sequence (length 12)
    last = off[b + 1] - 1
    q2, k2, v2 = q.copy(), k.copy(), v.copy()
    q2[last] += 1.0; k2[last] -= 2.0; v2[last] *= 3.0
    spec.timestamps = spec.timestamps.copy(); spec.timestamps[last] += 10**6
    A2 = O.attention_forward(off, 2, 3, q2, k2, v2, spec)
    assert np.array_equal(np.delete(A2, last, axis=0), np.delete(A, last, axis=0))


def test_v_rows_outside_allowed_set_irrelevant():
    # for query q, permuting V rows outside its allowed set leaves A[q] unchanged
    off = np.array([0, 20]); r = np.random.default_rng(9)
    q, k, v = (r.standard_normal((20, 4)) for _ in range(3))
    spec = O.AttnSpec(K1=3, K2=2, N=4.0)
    A = O.attention_forward(off, 1, 4, q, k, v, spec)
    qi = 15  # allowed keys: 0,1 (global) and 12..15 (band)
    outside = [j for j in range(20) if not (j < 2 or 12 <= j <= 15)]
    v2 = v.copy(); v2[outside] = v[outside][::-1] * 7.0
    A2 = O.attention_forward(off, 1, 4, q, k, v2, spec)
    assert np.array_equal(A2[qi], A[qi])


def test_small_score_limit_is_masked_matmul():
    # silu(s) = s/2 + s^2/4 + O(s^4): with tiny scores A -> (1/2N)((alpha Q K^T) (.) M) V,
    # a textbook masked matmul; error bounded by the s^2/4 term.
    off = np.array([0, 30]); r = np.random.default_rng(4)
    eps = 1e-4
    q, k, v = r.standard_normal((30, 4)) * eps, r.standard_normal((30, 4)), r.standard_normal((30, 4))
    spec = O.AttnSpec(K1=5, K2=3, alpha=1.0, N=2.0)
    A = O.attention_forward(off, 1, 4, q, k, v, spec)
    M = dense_mask(30, 5, 3)
    lin = ((q @ k.T) * M) @ v / (2 * spec.N)
    smax = np.max(np.abs(q @ k.T))
    assert np.max(np.abs(A - lin)) <= (smax ** 2 / 4 / spec.N) * np.max(np.abs(v).sum(0)) * 30 + 1e-18
    assert np.max(np.abs(A - lin)) < 1e-3 * np.max(np.abs(lin))


# ---------------------------------------------------------------------------
# attention backward: central finite differences
# ---------------------------------------------------------------------------
def test_attention_backward_finite_differences():
    off, q, k, v, spec = small_case(lengths=(5, 7), rab=True)
    r = np.random.default_rng(1)
    dA = r.standard_normal(q.shape)
    (dQ, dK, dV, dpos, dts), work = O.attention_backward(off, 2, 3, q, k, v, dA, spec, return_work=True)
    assert work == 2 * (closed_form_nnz(5, 2, 1) + closed_form_nnz(7, 2, 1))

    def loss(q_, k_, v_, pos_, ts_):
        s2 = O.AttnSpec(spec.K1, spec.K2, spec.alpha, spec.N, pos_, ts_, spec.timestamps)
        return float(np.sum(O.attention_forward(off, 2, 3, q_, k_, v_, s2) * dA))

    h = 1e-6
    args = [q, k, v, spec.pos_w, spec.ts_w]
    grads = [dQ, dK, dV, dpos, dts]
    for ai, (a, g) in enumerate(zip(args, grads)):
        fd = np.zeros_like(a)
        for idx in np.ndindex(a.shape):
            ap, am = [x.copy() for x in args], [x.copy() for x in args]
            ap[ai][idx] += h; am[ai][idx] -= h
            fd[idx] = (loss(*ap) - loss(*am)) / (2 * h)
        assert rel_inf(g, fd) < 1e-6, ai


# ---------------------------------------------------------------------------
# LayerNorm / SiLU against library routines
# ---------------------------------------------------------------------------
def test_silu_and_grad():
    assert O.silu(np.array(0.0)) == 0.0
    assert abs(O.silu(np.array(20.0)) - 20.0) < 1e-7
    x = torch.tensor([-2.0, -0.5, 1.3, 4.0], dtype=torch.float64, requires_grad=True)
    torch.nn.functional.silu(x).sum().backward()
    assert np.allclose(O.silu(x.detach().numpy()), torch.nn.functional.silu(x).detach().numpy(), atol=1e-15)
    assert np.allclose(O.silu_grad(x.detach().numpy()), x.grad.numpy(), atol=1e-14)


def test_layer_norm_vs_torch():
    r = np.random.default_rng(2)
    x = r.standard_normal((7, 10)); w = 1 + 0.1 * r.standard_normal(10); b = 0.1 * r.standard_normal(10)
    g = r.standard_normal((7, 10))
    y, mu, rs = O.layer_norm(x, w, b, 1e-6)
    xt = torch.tensor(x, requires_grad=True); wt = torch.tensor(w, requires_grad=True); bt = torch.tensor(b, requires_grad=True)
    yt = torch.nn.functional.layer_norm(xt, (10,), wt, bt, eps=1e-6)
    (yt * torch.tensor(g)).sum().backward()
    assert np.max(np.abs(y - yt.detach().numpy())) < 1e-13
    dx, dw, db = O.layer_norm_backward(g, x, mu, rs, w)
    assert np.max(np.abs(dx - xt.grad.numpy())) < 1e-12
    assert np.max(np.abs(dw - wt.grad.numpy())) < 1e-12
    assert np.max(np.abs(db - bt.grad.numpy())) < 1e-12
    # constant row -> bias
    yc, _, _ = O.layer_norm(np.full((1, 10), 3.0), w, b, 1e-6)
    assert np.allclose(yc[0], b, atol=1e-12)


# ---------------------------------------------------------------------------
# the layer (Eqs. 1-5, Listing 1)
# ---------------------------------------------------------------------------
def small_layer(seed=0, lengths=(5, 7), H=2, dh=3, rab=True, K1=2, K2=1):
    cfg = synth.Config("t", list(lengths), H=H, dh=dh, K1=K1, K2=K2, N=9.0, seed=seed)
    r = np.random.default_rng(seed)
    d = H * dh
    p = synth.layer_params(d, seed)
    prm = O.LayerParams(**{k_: np.asarray(v_, np.float64) for k_, v_ in p.items()})
    x = r.standard_normal((cfg.T, d))
    spec = O.AttnSpec(K1=K1, K2=K2, alpha=0.8, N=9.0)
    if rab:
        spec.pos_w = r.standard_normal(8) * 0.5
        spec.ts_w = r.standard_normal(6) * 0.5
        spec.timestamps = synth.timestamps(seed, lengths)
    return cfg, prm, x, spec


def test_layer_zero_weights_is_identity():
    cfg, prm, x, spec = small_layer()
    prm.w1 = 0 * prm.w1; prm.w2 = 0 * prm.w2; prm.b1 = 0 * prm.b1; prm.b2 = 0 * prm.b2
    out, _ = O.layer_forward(x, cfg.offsets(), prm, cfg.H, spec)
    assert np.array_equal(out, x)


def torch_dense_layer(x, off, prm, H, alpha, N, eps):
    """Full-causal, rab-free layer as dense torch fp64 ops (autograd gives gradients)."""
    d = x.shape[1]; dh = d // H
    t = {k_: torch.tensor(getattr(prm, k_), requires_grad=True) for k_ in
         ("ln1_w", "ln1_b", "w1", "b1", "ln2_w", "ln2_b", "w2", "b2")}
    X = torch.tensor(x, requires_grad=True)
    xh = torch.nn.functional.layer_norm(X, (d,), t["ln1_w"], t["ln1_b"], eps=eps)
    s = torch.nn.functional.silu(xh @ t["w1"] + t["b1"])
    U, V, Q, K = s.split(d, dim=1)
    outs = []
    for b in range(len(off) - 1):
        o0, o1 = int(off[b]), int(off[b + 1]); L = o1 - o0
        M = torch.tril(torch.ones(L, L, dtype=torch.bool))
        heads = []
        for h in range(H):
            sl = slice(h * dh, (h + 1) * dh)
            S = alpha * Q[o0:o1, sl] @ K[o0:o1, sl].T
            P_ = torch.where(M, torch.nn.functional.silu(S) / N, torch.zeros_like(S))
            heads.append(P_ @ V[o0:o1, sl])
        outs.append(torch.cat(heads, dim=1))
    A = torch.cat(outs, dim=0)
    Y = torch.nn.functional.layer_norm(A, (d,), t["ln2_w"], t["ln2_b"], eps=eps) * U
    out = Y @ t["w2"] + t["b2"] + X
    return out, X, t


def test_layer_vs_torch_autograd_full_causal():
    cfg, prm, x, spec = small_layer(rab=False, lengths=(6, 9, 4), K1=O.FULL, K2=0)
    out, cache = O.layer_forward(x, cfg.offsets(), prm, cfg.H, spec)
    tout, X, t = torch_dense_layer(x, cfg.offsets(), prm, cfg.H, spec.alpha, spec.N, prm.eps)
    assert rel_inf(out, tout.detach().numpy()) < 1e-13
    dout = np.random.default_rng(7).standard_normal(out.shape)
    (tout * torch.tensor(dout)).sum().backward()
    dx, g = O.layer_backward(dout, cfg.offsets(), prm, cfg.H, spec, cache=cache)
    assert rel_inf(dx, X.grad.numpy()) < 1e-12
    for k_ in t:
        assert rel_inf(g[k_], t[k_].grad.numpy()) < 1e-11, k_


def test_layer_backward_finite_differences():
    cfg, prm, x, spec = small_layer(rab=True)
    dout = np.random.default_rng(8).standard_normal(x.shape)
    dx, g = O.layer_backward(dout, cfg.offsets(), prm, cfg.H, spec, x=x)

    def loss(x_, prm_, spec_):
        out, _ = O.layer_forward(x_, cfg.offsets(), prm_, cfg.H, spec_)
        return float(np.sum(out * dout))

    h = 1e-6
    rng = np.random.default_rng(0)

    def fd_check(get, set_, grad, n_probe=12):
        base = get().copy()
        idxs = [tuple(rng.integers(0, s) for s in base.shape) for _ in range(n_probe)]
        for idx in idxs:
            a = base.copy(); a[idx] += h; set_(a); lp = loss(x_c[0], prm, spec)
            a = base.copy(); a[idx] -= h; set_(a); lm = loss(x_c[0], prm, spec)
            set_(base)
            fd = (lp - lm) / (2 * h)
            assert abs(grad[idx] - fd) <= 1e-6 * max(1.0, np.max(np.abs(grad))), (idx, grad[idx], fd)

    x_c = [x]
    fd_check(lambda: x_c[0], lambda a: x_c.__setitem__(0, a), dx)
    for name in ("ln1_w", "ln1_b", "w1", "b1", "ln2_w", "ln2_b", "w2", "b2"):
        fd_check(lambda n=name: getattr(prm, n), lambda a, n=name: setattr(prm, n, a), g[name])
    fd_check(lambda: spec.pos_w, lambda a: setattr(spec, "pos_w", a), g["pos_w"])
    fd_check(lambda: spec.ts_w, lambda a: setattr(spec, "ts_w", a), g["ts_w"])


# ---------------------------------------------------------------------------
# partitioner oracle (LPT)
# ---------------------------------------------------------------------------
def test_seq_cost_counts_the_step_flops():
    """seq_cost against an independent count: the layer step's GEMM list written out from
    their shapes (M x N x K, 2 flops per multiply-add)
    plus 4 d_h (forward) + 10 d_h (backward, S recomputed) flops per allowed pair and head,
    the pairs counted by brute force on the dense mask (never the closed form)."""
    for L, d, H, K1, K2 in [(1, 64, 2, 16, 2), (17, 64, 2, 16, 2), (300, 128, 1, 40, 7), (97, 256, 2, 0, 0),
                            (64, 64, 2, O.FULL, 0), (257, 64, 4, 128, 129)]:
        gemms = [(L, 4 * d, d),      # F2: h = x^ W1
                 (L, d, d),          # F7: Y W2
                 (L, 4 * d, d),      # B3: remat h = x^ W1
                 (L, d, d),          # B1: dY = dOut W2^T
                 (d, d, L),          # B1: dW2 = Y^T dOut
                 (d, 4 * d, L),      # B5: dW1 = x^T dH
                 (L, d, 4 * d)]      # B5: dx^ = dH W1^T
        gemm_flops = sum(2 * M * N * K for M, N, K in gemms)
        q = np.arange(L)[:, None]
        k = np.arange(L)[None, :]
        win = np.ones((L, L), bool) if K1 == O.FULL else (q - k <= K1)
        pairs = int(((k <= q) & (win | (k < K2))).sum())
        assert O.seq_cost(L, d, H, K1, K2) == gemm_flops + pairs * H * (4 + 10) * (d // H)


def test_partition_lpt_properties():
    import itertools
    lengths = [300, 17, 1000, 1000, 64, 512, 999, 3, 250]
    owner, load = O.partition_lpt(lengths, 3, d=64, H=2, K1=16, K2=2)
    assert sorted(set(owner)) == [0, 1, 2] and len(owner) == len(lengths)
    costs = [O.seq_cost(L, 64, 2, 16, 2) for L in lengths]
    for r in range(3):
        assert abs(load[r] - sum(c for c, o in zip(costs, owner) if o == r)) < 1e-6 * sum(costs)
    # Graham's LPT bound against the brute-force optimum
    best = min(max(sum(c for c, a in zip(costs, asg) if a == r) for r in range(3))
               for asg in itertools.product(range(3), repeat=len(lengths)))
    assert max(load) <= (4 / 3 - 1 / 9) * best + 1e-9
    assert O.partition_lpt(lengths, 3, 64, 2, 16, 2) == (owner, load)


def test_rab_gradient_absolute_sums():
    """The |ds| sums beside d pos_bias / d time_bias (R15b): never below |sum|, equal to it for a
    single pair, unchanged when dA flips sign (the sums flip), and both tables add up the same
    sum of |ds| over all visible pairs (every pair lands in exactly one entry of each)."""
    cfg = synth.Config("abs", [1, 9, 30], H=2, dh=4, K1=5, K2=2, N=30.0, seed=8, pos_len=12, ts_len=8)
    q, k, v, dA = synth.attn_inputs(cfg)
    pos, ts = synth.rab_tables(cfg)
    t = synth.timestamps(cfg.seed, cfg.lengths)
    spec = O.AttnSpec(K1=cfg.K1, K2=cfg.K2, alpha=1.0, N=cfg.N, pos_w=pos, ts_w=ts, timestamps=t)
    r = O.attention_backward(cfg.offsets(), cfg.H, cfg.dh, q, k, v, dA, spec, return_abs=True)
    dpos, dts, apos, ats = r[3], r[4], r[5], r[6]
    assert np.all(apos >= np.abs(dpos) - 1e-15) and np.all(ats >= np.abs(dts) - 1e-15)
    assert abs(apos.sum() - ats.sum()) <= 1e-12 * ats.sum()
    n = O.attention_backward(cfg.offsets(), cfg.H, cfg.dh, q, k, v, -dA, spec, return_abs=True)
    assert np.allclose(n[3], -dpos, atol=1e-15) and np.allclose(n[5], apos, rtol=1e-12) and np.allclose(n[6], ats, rtol=1e-12)
    one = synth.Config("one", [1], H=1, dh=4, K1=0, K2=0, N=1.0, seed=9, pos_len=3, ts_len=4)
    q1, k1, v1, d1 = synth.attn_inputs(one)
    s1 = O.AttnSpec(K1=0, K2=0, alpha=1.0, N=1.0, pos_w=pos[:3], ts_w=ts[:4], timestamps=t[:1])
    r1 = O.attention_backward(one.offsets(), 1, 4, q1, k1, v1, d1, s1, return_abs=True)
    assert r1[5][0] == abs(r1[3][0]) and r1[6][0] == abs(r1[4][0])
