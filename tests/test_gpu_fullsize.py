"""GPU parity at BASELINE.json's full size (cfg3: 16 x 16384 tokens, 4 x 128 heads, SLA
window 1024 + 128 global, rab on with P = 16384), in the launch configuration bench.py times
(the whole batch through one call).  Sequences are independent and N is explicit (DESIGN.md
R5), so the rows of a sampled sequence must equal the oracle run on that sequence alone; those
rows are compared element by element (per-tensor infinity-norm relative, bf16 bar 2e-2).
Batch-level sums (parameter / rab gradients) are compared on two full 16384-token sequences."""
import numpy as np
import pytest
import torch

import oracle as O
from gpu_util import rel_inf, to_dev, to_np
from paper_2602_16986_b200 import synth
from paper_2602_16986_b200 import uhstu as U

pytestmark = pytest.mark.gpu

TOL = 2e-2
SAMPLE = 7          # sampled sequence (of 16)


def _cfg3():
    return synth.config("cfg3")


def _spec_one(cfg, pos, ts, t_one):
    return O.AttnSpec(K1=cfg.K1, K2=cfg.K2, alpha=cfg.alpha, N=float(cfg.N), pos_w=pos, ts_w=ts, timestamps=t_one)


def test_attention_cfg3_full_size_sampled_sequence():
    cfg = _cfg3()
    off = cfg.offsets()
    q, k, v, dA = synth.attn_inputs(cfg)
    pos, ts = synth.rab_tables(cfg)
    t = synth.timestamps(cfg.seed, cfg.lengths)
    d = cfg.d
    buf = torch.empty(cfg.T, 4 * d, dtype=torch.bfloat16, device="cuda")   # U|V|Q|K like the layer's
    buf[:, d:2 * d] = to_dev(v, U.BF16)
    buf[:, 2 * d:3 * d] = to_dev(q, U.BF16)
    buf[:, 3 * d:] = to_dev(k, U.BF16)
    jag = U.JaggedBatch(off)
    attn = U.Attn(cfg.H, cfg.dh, cfg.alpha, float(cfg.N), torch.from_numpy(pos).cuda(), torch.from_numpy(ts).cuda(),
                  torch.from_numpy(t).cuda())
    m = U.mask(cfg.K1, cfg.K2)
    A = U.attn_fwd(jag, m, attn, buf[:, 2 * d:3 * d], buf[:, 3 * d:], buf[:, d:2 * d])
    dq, dk, dv, _, _ = U.attn_bwd(jag, m, attn, buf[:, 2 * d:3 * d], buf[:, 3 * d:], buf[:, d:2 * d],
                                  to_dev(dA, U.BF16))
    torch.cuda.synchronize()
    r0, r1 = int(off[SAMPLE]), int(off[SAMPLE + 1])
    rows = slice(r0, r1)
    one = np.array([0, r1 - r0], np.int32)
    spec = _spec_one(cfg, pos, ts, t[rows])
    ref_a = O.attention_forward(one, cfg.H, cfg.dh, q[rows], k[rows], v[rows], spec)
    assert rel_inf(to_np(A[rows]), ref_a) <= TOL
    ref = O.attention_backward(one, cfg.H, cfg.dh, q[rows], k[rows], v[rows], dA[rows], spec)
    for name, got, r in zip(("dQ", "dK", "dV"), (dq, dk, dv), ref[:3]):
        e = rel_inf(to_np(got[rows]), r)
        assert e <= TOL, (name, e)


def test_layer_cfg3_full_size_sampled_sequence():
    cfg = _cfg3()
    off = cfg.offsets()
    p = synth.layer_params(cfg.d, cfg.seed)
    x, dout = synth.layer_inputs(cfg)
    pos, ts = synth.rab_tables(cfg)
    t = synth.timestamps(cfg.seed, cfg.lengths)
    f = lambda a: torch.from_numpy(a).cuda()
    w = lambda a: torch.from_numpy(a).to("cuda", torch.bfloat16)
    prm = U.Params(f(p["ln1_w"]), f(p["ln1_b"]), w(p["w1"]), f(p["ln2_w"]), f(p["ln2_b"]), w(p["w2"]),
                   f(p["b1"]), f(p["b2"]))
    attn = U.Attn(cfg.H, cfg.dh, cfg.alpha, float(cfg.N), f(pos), f(ts), f(t))
    jag = U.JaggedBatch(off)
    m = U.mask(cfg.K1, cfg.K2)
    X = to_dev(x, U.BF16)
    out, saved = U.layer_fwd(jag, m, prm, attn, X)
    dx, _ = U.layer_bwd(jag, m, prm, attn, X, saved, to_dev(dout, U.BF16))
    torch.cuda.synchronize()
    r0, r1 = int(off[SAMPLE]), int(off[SAMPLE + 1])
    rows = slice(r0, r1)
    one = np.array([0, r1 - r0], np.int32)
    prm_o = O.LayerParams(**{kk: np.asarray(vv, np.float64) for kk, vv in p.items()})
    spec = _spec_one(cfg, pos, ts, t[rows])
    ref_out, cache = O.layer_forward(x[rows], one, prm_o, cfg.H, spec)
    assert rel_inf(to_np(out[rows]), ref_out) <= TOL
    ref_dx, _ = O.layer_backward(dout[rows], one, prm_o, cfg.H, spec, cache=cache)
    assert rel_inf(to_np(dx[rows]), ref_dx) <= TOL


def test_attention_cfg2_full_size_sampled_sequences():
    """cfg2 (BASELINE configs[1]): 32 sequences of U[1024, 4096] tokens, full causal, rab on."""
    cfg = synth.config("cfg2")
    off = cfg.offsets()
    q, k, v, dA = synth.attn_inputs(cfg)
    pos, ts = synth.rab_tables(cfg)
    t = synth.timestamps(cfg.seed, cfg.lengths)
    d = cfg.d
    buf = torch.empty(cfg.T, 4 * d, dtype=torch.bfloat16, device="cuda")
    buf[:, d:2 * d] = to_dev(v, U.BF16)
    buf[:, 2 * d:3 * d] = to_dev(q, U.BF16)
    buf[:, 3 * d:] = to_dev(k, U.BF16)
    jag = U.JaggedBatch(off)
    attn = U.Attn(cfg.H, cfg.dh, cfg.alpha, float(cfg.N), torch.from_numpy(pos).cuda(), torch.from_numpy(ts).cuda(),
                  torch.from_numpy(t).cuda())
    m = U.mask(cfg.K1, cfg.K2)
    Q, K, V = buf[:, 2 * d:3 * d], buf[:, 3 * d:], buf[:, d:2 * d]
    A = U.attn_fwd(jag, m, attn, Q, K, V)
    dq, dk, dv, _, _ = U.attn_bwd(jag, m, attn, Q, K, V, to_dev(dA, U.BF16))
    torch.cuda.synchronize()
    longest = int(np.argmax(cfg.lengths))
    for b in sorted({longest, 5}):
        r0, r1 = int(off[b]), int(off[b + 1])
        rows = slice(r0, r1)
        one = np.array([0, r1 - r0], np.int32)
        spec = O.AttnSpec(K1=O.FULL, K2=0, alpha=cfg.alpha, N=float(cfg.N), pos_w=pos, ts_w=ts, timestamps=t[rows])
        assert rel_inf(to_np(A[rows]), O.attention_forward(one, cfg.H, cfg.dh, q[rows], k[rows], v[rows], spec)) <= TOL
        ref = O.attention_backward(one, cfg.H, cfg.dh, q[rows], k[rows], v[rows], dA[rows], spec)
        for name, got, r in zip(("dQ", "dK", "dV"), (dq, dk, dv), ref[:3]):
            e = rel_inf(to_np(got[rows]), r)
            assert e <= TOL, (b, name, e)


def test_layer_cfg3_two_sequences_all_gradients():
    """Parameter and rab gradients at the cfg3 shape (4 x 128 heads, SLA 1024 + 128 global,
    P = 16384, N = 16384) on two full 16384-token sequences through one call -- the launch
    configuration of bench.py at 1/8 of its batch: the split-K weight-gradient atomics, the fused
    bias column sums and the per-CTA d rab reductions all run at full sequence length.  Every
    gradient (and out, dx) against the oracle."""
    full = _cfg3()
    cfg = synth.Config("cfg3x2", [16384, 16384], H=full.H, dh=full.dh, K1=full.K1, K2=full.K2, N=full.N,
                       seed=full.seed)
    assert cfg.P == 16384
    p = synth.layer_params(cfg.d, cfg.seed)
    x, dout = synth.layer_inputs(cfg)
    pos, ts = synth.rab_tables(cfg)
    t = synth.timestamps(cfg.seed, cfg.lengths)
    f = lambda a: torch.from_numpy(a).cuda()
    w = lambda a: torch.from_numpy(a).to("cuda", torch.bfloat16)
    prm = U.Params(f(p["ln1_w"]), f(p["ln1_b"]), w(p["w1"]), f(p["ln2_w"]), f(p["ln2_b"]), w(p["w2"]),
                   f(p["b1"]), f(p["b2"]))
    attn = U.Attn(cfg.H, cfg.dh, cfg.alpha, float(cfg.N), f(pos), f(ts), f(t))
    jag = U.JaggedBatch(cfg.offsets())
    m = U.mask(cfg.K1, cfg.K2)
    X = to_dev(x, U.BF16)
    out, saved = U.layer_fwd(jag, m, prm, attn, X)
    dx, g = U.layer_bwd(jag, m, prm, attn, X, saved, to_dev(dout, U.BF16))
    torch.cuda.synchronize()
    prm_o = O.LayerParams(**{kk: np.asarray(vv, np.float64) for kk, vv in p.items()})
    spec = O.AttnSpec(K1=cfg.K1, K2=cfg.K2, alpha=cfg.alpha, N=float(cfg.N), pos_w=pos, ts_w=ts, timestamps=t)
    ref_out, cache = O.layer_forward(x, cfg.offsets(), prm_o, cfg.H, spec)
    ref_dx, ref_g = O.layer_backward(dout, cfg.offsets(), prm_o, cfg.H, spec, cache=cache, rab_abs=True)
    assert rel_inf(to_np(out), ref_out) <= TOL
    assert rel_inf(to_np(dx), ref_dx) <= TOL
    for k in ("ln1_w", "ln1_b", "w1", "b1", "ln2_w", "ln2_b", "w2", "b2"):
        e = rel_inf(to_np(g[k]), ref_g[k])
        assert e <= TOL, (k, e)
    # d pos_bias / d time_bias sum ds of both signs over up to millions of pairs per entry, so
    # |sum| can be orders of magnitude below the sum of |terms|; the bar applies to the latter,
    # the scale of the summation error bound (R15b): |g - r| <= TOL * sum |ds| per entry
    for k, ok in (("pos_bias", "pos_w"), ("time_bias", "ts_w")):
        err = np.abs(to_np(g[k]) - ref_g[ok])
        assert np.all(err <= TOL * ref_g[ok + "_abs"] + 1e-12), (k, float(np.max(err / (ref_g[ok + "_abs"] + 1e-30))))
