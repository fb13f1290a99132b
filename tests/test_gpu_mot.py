"""NEXT-4: Mixture of Transducers on the GPU against oracle/mot.py.

* the fusion alone (uh_mot_fuse_fwd / _bwd on given branch states; oracle branches with no
  layers), ragged users, 2 and 3 branches, d = 128 (column-sum pass) and d = 256 (column sums
  fused into the split-K dW_f GEMM), fp32 and bf16; the zero rows of dX_k are checked
  bit-exact (R30), everything else per tensor at the dtype's bar;
* a whole MoT step (two branch stacks of different depth and mask over the same users, the
  fusion, the backward into every bucket) against mot_forward / mot_backward in fp64."""
import numpy as np
import pytest
import torch

import mot as M
import oracle as O
from gpu_util import rel_inf, tdt, to_dev, to_np
from paper_2602_16986_b200 import dist as D
from paper_2602_16986_b200 import mot as GM
from paper_2602_16986_b200 import synth
from paper_2602_16986_b200 import uhstu as U

pytestmark = pytest.mark.gpu

TOL = {U.BF16: 2e-2, U.F32: 1e-4}


def _offsets(lengths):
    off = np.zeros(len(lengths) + 1, np.int32)
    off[1:] = np.cumsum(lengths)
    return off


@pytest.mark.parametrize("dt", [U.BF16, U.F32])
@pytest.mark.parametrize("K,d,n_cand", [(2, 128, 3), (3, 256, 1), (2, 256, 5)])
def test_fusion_matches_oracle(dt, K, d, n_cand):
    B = 37                                             # C = B n_cand: ragged against the 128-row tiles
    r = np.random.default_rng(K * 1000 + d + n_cand)
    lens = [synth.mot_lengths(7, B, n_cand, 90, k) for k in range(K)]
    offs = [_offsets(l) for l in lens]
    xs = [synth.round_bf16(r.standard_normal((int(o[-1]), d)).astype(np.float32)) for o in offs]
    W, bias = synth.mot_params(d, K, 11)
    dE = synth.round_bf16(r.standard_normal((B * n_cand, d)).astype(np.float32))
    brs = [M.Branch(x=x, offsets=o, layers=[]) for x, o in zip(xs, offs)]
    E_ref, cache = M.mot_forward(brs, n_cand, W, bias)
    dxs_ref, _, dW_ref, db_ref = M.mot_backward(dE, brs, n_cand, W, bias, cache=cache)

    jags = [U.JaggedBatch(o) for o in offs]
    X = [to_dev(x, dt) for x in xs]
    Wd, bd = to_dev(W, dt), torch.from_numpy(bias).cuda()
    E = U.mot_fuse_fwd(jags, X, n_cand, Wd, bd)
    dW = torch.full((K * d, d), 7.0, device="cuda")       # overwritten (accumulate = 0)
    db = torch.full((d,), 7.0, device="cuda")
    dxs = [torch.full_like(x, 3.0) for x in X]             # every row written
    U.mot_fuse_bwd(jags, X, n_cand, Wd, to_dev(dE, dt), dW, db, dxs=dxs)
    torch.cuda.synchronize()
    tol = TOL[dt]
    assert rel_inf(to_np(E), E_ref) <= tol
    assert rel_inf(to_np(dW), dW_ref) <= tol
    assert rel_inf(to_np(db), db_ref) <= tol
    for k in range(K):
        got, ref = to_np(dxs[k]), dxs_ref[k]
        cand = M.candidate_rows(offs[k], n_cand)
        other = np.setdiff1d(np.arange(got.shape[0]), cand)
        assert np.all(got[other] == 0.0)
        assert rel_inf(got[cand], ref[cand]) <= tol
    # accumulate = 1 adds the same gradients again
    U.mot_fuse_bwd(jags, X, n_cand, Wd, to_dev(dE, dt), dW, db, accumulate=True, dxs=dxs)
    torch.cuda.synchronize()
    assert rel_inf(to_np(dW), 2 * dW_ref) <= tol
    assert rel_inf(to_np(db), 2 * db_ref) <= tol


def test_fusion_identical_branches_selector():
    """W_f = [I; 0] returns branch 0's candidate rows exactly (bf16 states, bf16 identity)."""
    B, n_cand, d = 20, 4, 128
    lens = synth.mot_lengths(3, B, n_cand, 60, 0)
    off = _offsets(lens)
    x = synth.round_bf16(np.random.default_rng(2).standard_normal((int(off[-1]), d)).astype(np.float32))
    jag = U.JaggedBatch(off)
    X = to_dev(x, U.BF16)
    sel = np.concatenate([np.eye(d), np.zeros((d, d))], axis=0).astype(np.float32)
    E = U.mot_fuse_fwd([jag, jag], [X, X * 2], n_cand, to_dev(sel, U.BF16), None)
    torch.cuda.synchronize()
    assert np.array_equal(to_np(E), x[M.candidate_rows(off, n_cand)])


def _layer(p, H, dh, attn_args, m):
    f = lambda a: torch.from_numpy(a).cuda()
    w = lambda a: torch.from_numpy(a).to("cuda", torch.bfloat16)
    prm = U.Params(f(p["ln1_w"]), f(p["ln1_b"]), w(p["w1"]), f(p["ln2_w"]), f(p["ln2_b"]), w(p["w2"]),
                   f(p["b1"]), f(p["b2"]))
    return prm, U.Attn(H, dh, 1.0, *attn_args)


def test_mot_step_matches_oracle():
    """Two transducers over the same 9 users: a 2-layer SLA branch with rab ("C-seq", longer)
    and a 1-layer full-causal branch ("E-seq", shorter), n_cand = 4 candidates per user."""
    B, n_cand, H, dh = 9, 4, 1, 128
    d = H * dh
    specs = [dict(lo=150, hi=420, layers=2, K1=64, K2=8, N=420.0, seed=21),
             dict(lo=40, hi=160, layers=1, K1=None, K2=0, N=160.0, seed=22)]
    W, bias = synth.mot_params(d, 2, 5)
    r = np.random.default_rng(1)
    dE = synth.round_bf16(r.standard_normal((B * n_cand, d)).astype(np.float32))
    brs_o, stacks, xs = [], [], []
    for k, s in enumerate(specs):
        lens = synth.mot_lengths(s["seed"], B, s["lo"], s["hi"], k)
        cfg = synth.Config(f"mot{k}", lens, H=H, dh=dh, K1=s["K1"] or 1, K2=s["K2"], N=s["N"], seed=s["seed"],
                           pos_len=96)
        off = cfg.offsets()
        x, _ = synth.layer_inputs(cfg)
        pos, ts = synth.rab_tables(cfg)
        t = synth.timestamps(cfg.seed, lens)
        params = [synth.layer_params(d, s["seed"], layer=l) for l in range(s["layers"])]
        K1o = O.FULL if s["K1"] is None else s["K1"]
        layers_o = []
        for p in params:
            prm = O.LayerParams(**{kk: np.asarray(v, np.float64) for kk, v in p.items()})
            layers_o.append((prm, H, O.AttnSpec(K1=K1o, K2=s["K2"], alpha=1.0, N=s["N"], pos_w=pos, ts_w=ts,
                                                timestamps=t)))
        brs_o.append(M.Branch(x=x, offsets=off, layers=layers_o))
        f = lambda a: torch.from_numpy(a).cuda()
        m = U.mask() if s["K1"] is None else U.mask(s["K1"], s["K2"])
        X = to_dev(x, U.BF16)
        layers = [_layer(p, H, dh, (s["N"], f(pos), f(ts), f(t)), m) for p in params]
        stacks.append(D.Stack(U.JaggedBatch(off), m, layers, X))
        xs.append(X)
    E_ref, cache = M.mot_forward(brs_o, n_cand, W, bias)
    dxs_ref, grads_ref, dW_ref, db_ref = M.mot_backward(dE, brs_o, n_cand, W, bias, cache=cache)

    mot = GM.MoT(stacks, n_cand, to_dev(W, U.BF16), torch.from_numpy(bias).cuda())
    E = mot.forward(xs)
    dxs, handles = mot.backward(xs, to_dev(dE, U.BF16))
    torch.cuda.synchronize()
    assert not handles                                   # single process: nothing to all-reduce
    TOLB = 2e-2
    assert rel_inf(to_np(E), E_ref) <= TOLB
    assert rel_inf(to_np(mot.bucket.views["w_f"]), dW_ref) <= TOLB
    assert rel_inf(to_np(mot.bucket.views["b_f"]), db_ref) <= TOLB
    for k in range(2):
        assert rel_inf(to_np(dxs[k]), dxs_ref[k]) <= TOLB, k
        for l, g_ref in enumerate(grads_ref[k]):
            views = stacks[k].buckets[l].views
            for name in ("w1", "w2", "ln1_w", "b1"):
                e = rel_inf(to_np(views[name]), g_ref[name])
                assert e <= TOLB, (k, l, name, e)


@pytest.mark.parametrize("K,B,n_cand", [(8, 3, 2), (1, 1, 7)])
def test_fusion_edge_shapes(K, B, n_cand):
    """The branch limit (8), a single branch, a single user and n_cand equal to a whole sequence."""
    d = 128
    r = np.random.default_rng(K * 10 + B)
    lens = [[n_cand] + synth.mot_lengths(9, B - 1, n_cand, 40, k) for k in range(K)]
    offs = [_offsets(l) for l in lens]
    xs = [synth.round_bf16(r.standard_normal((int(o[-1]), d)).astype(np.float32)) for o in offs]
    W, bias = synth.mot_params(d, K, 13)
    dE = synth.round_bf16(r.standard_normal((B * n_cand, d)).astype(np.float32))
    brs = [M.Branch(x=x, offsets=o, layers=[]) for x, o in zip(xs, offs)]
    E_ref, cache = M.mot_forward(brs, n_cand, W, bias)
    dxs_ref, _, dW_ref, db_ref = M.mot_backward(dE, brs, n_cand, W, bias, cache=cache)
    jags = [U.JaggedBatch(o) for o in offs]
    X = [to_dev(x, U.BF16) for x in xs]
    Wd, bd = to_dev(W, U.BF16), torch.from_numpy(bias).cuda()
    E = U.mot_fuse_fwd(jags, X, n_cand, Wd, bd)
    dW = torch.empty(K * d, d, device="cuda")
    db = torch.empty(d, device="cuda")
    dxs = U.mot_fuse_bwd(jags, X, n_cand, Wd, to_dev(dE, U.BF16), dW, db)
    torch.cuda.synchronize()
    assert rel_inf(to_np(E), E_ref) <= 2e-2
    assert rel_inf(to_np(dW), dW_ref) <= 2e-2 and rel_inf(to_np(db), db_ref) <= 2e-2
    for k in range(K):
        assert rel_inf(to_np(dxs[k]), dxs_ref[k]) <= 2e-2
