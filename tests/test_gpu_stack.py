"""NEXT-1: the inference schedule with attention truncation — SLA layers on
the whole jagged sequences, then the latest L' tokens of each sequence (uh_jagged_slice_latest,
P:198-199) through full-causal layers — against the oracle composed layer by layer
(numpy slicing of the oracle's own rows and timestamps).  bf16 bar 2e-2 per tensor."""
import numpy as np
import pytest
import torch

import oracle as O
from gpu_util import rel_inf, to_dev, to_np
from paper_2602_16986_b200 import stack as S
from paper_2602_16986_b200 import synth
from paper_2602_16986_b200 import uhstu as U

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("l_keep", [256, 64])
def test_truncated_inference_stack(l_keep):
    lengths = [300, 700, 1200, 64, 5]
    H, dh = 2, 128
    d = H * dh
    n_full, n_trunc = 2, 2
    K1, K2, N_full = 128, 16, 1200.0
    cfg = synth.Config("stack", lengths, H=H, dh=dh, K1=K1, K2=K2, N=N_full, seed=5, pos_len=64)
    x, _ = synth.layer_inputs(cfg)
    pos, ts = synth.rab_tables(cfg)
    t = synth.timestamps(cfg.seed, lengths)
    params = [synth.layer_params(d, cfg.seed, layer=l) for l in range(n_full + n_trunc)]

    # ---- GPU: one call per layer through the C ABI
    f = lambda a: torch.from_numpy(a).cuda()
    w = lambda a: torch.from_numpy(a).to("cuda", torch.bfloat16)
    layers = []
    for l, p in enumerate(params):
        prm = U.Params(f(p["ln1_w"]), f(p["ln1_b"]), w(p["w1"]), f(p["ln2_w"]), f(p["ln2_b"]), w(p["w2"]),
                       f(p["b1"]), f(p["b2"]))
        attn = U.Attn(H, dh, 1.0, N_full, f(pos), f(ts), f(t))
        m = U.mask(K1, K2) if l < n_full else U.mask()
        layers.append(S.Layer(prm, attn, m))
    jag = U.JaggedBatch(cfg.offsets())
    out, jt = S.forward_truncated(jag, to_dev(x, U.BF16), layers, n_full, l_keep, norm_n_truncated=float(l_keep))
    torch.cuda.synchronize()

    # ---- oracle: the same schedule, layer by layer in fp64
    off = cfg.offsets()
    h = x.astype(np.float64)
    for l in range(n_full):
        prm = O.LayerParams(**{k: np.asarray(v, np.float64) for k, v in params[l].items()})
        spec = O.AttnSpec(K1=K1, K2=K2, alpha=1.0, N=N_full, pos_w=pos, ts_w=ts, timestamps=t)
        h, _ = O.layer_forward(h, off, prm, H, spec)
    keep = np.concatenate([np.arange(off[b + 1] - min(l_keep, L), off[b + 1]) for b, L in enumerate(lengths)])
    lk = [min(l_keep, L) for L in lengths]
    off2 = np.zeros(len(lk) + 1, np.int32)
    off2[1:] = np.cumsum(lk)
    assert list(jt.lengths) == lk
    h, t2 = h[keep], t[keep]
    for l in range(n_full, n_full + n_trunc):
        prm = O.LayerParams(**{k: np.asarray(v, np.float64) for k, v in params[l].items()})
        spec = O.AttnSpec(K1=O.FULL, K2=0, alpha=1.0, N=float(l_keep), pos_w=pos, ts_w=ts, timestamps=t2)
        h, _ = O.layer_forward(h, off2, prm, H, spec)
    assert rel_inf(to_np(out), h) <= 2e-2


def test_cfg4_like_stack_per_layer_against_oracle():
    """cfg4's shape at test size: log-uniform (long-tail) lengths through a 3-layer stack with
    independent weights.  Every layer is checked against the oracle given the GPU's own input
    and incoming gradient (teacher forcing); Stack.step reproduces the chain."""
    from paper_2602_16986_b200 import dist as D
    lengths = synth.lengths_loguniform_until(4, 32, 1500, 6000)
    H, dh, n_layers = 2, 128, 3
    d = H * dh
    cfg = synth.Config("stack4", lengths, H=H, dh=dh, K1=256, K2=32, N=1500.0, seed=4, pos_len=64)
    x, dout = synth.layer_inputs(cfg)
    pos, ts = synth.rab_tables(cfg)
    t = synth.timestamps(cfg.seed, lengths)
    f = lambda a: torch.from_numpy(a).cuda()
    w = lambda a: torch.from_numpy(a).to("cuda", torch.bfloat16)
    attn = U.Attn(H, dh, 1.0, cfg.N, f(pos), f(ts), f(t))
    m = U.mask(cfg.K1, cfg.K2)
    jag = U.JaggedBatch(cfg.offsets())
    params = [synth.layer_params(d, cfg.seed, layer=l) for l in range(n_layers)]
    prms = [U.Params(f(p["ln1_w"]), f(p["ln1_b"]), w(p["w1"]), f(p["ln2_w"]), f(p["ln2_b"]), w(p["w2"]),
                     f(p["b1"]), f(p["b2"])) for p in params]
    X, G = to_dev(x, U.BF16), to_dev(dout, U.BF16)
    # the chain, layer by layer through the C ABI
    hs, saved = [X], []
    for prm in prms:
        out, sv = U.layer_fwd(jag, m, prm, attn, hs[-1])
        hs.append(out)
        saved.append(sv)
    gs, grads = [None] * n_layers, [None] * n_layers
    g = G
    for l in range(n_layers - 1, -1, -1):
        dx, gr = U.layer_bwd(jag, m, prms[l], attn, hs[l], saved[l], g)
        gs[l], grads[l] = g, gr
        g = dx
    torch.cuda.synchronize()
    off = cfg.offsets()
    spec = O.AttnSpec(K1=cfg.K1, K2=cfg.K2, alpha=1.0, N=cfg.N, pos_w=pos, ts_w=ts, timestamps=t)
    for l in range(n_layers):
        prm_o = O.LayerParams(**{k: np.asarray(v, np.float64) for k, v in params[l].items()})
        ref_out, cache = O.layer_forward(to_np(hs[l]), off, prm_o, H, spec)
        assert rel_inf(to_np(hs[l + 1]), ref_out) <= 2e-2, ("out", l)
        ref_dx, ref_g = O.layer_backward(to_np(gs[l]), off, prm_o, H, spec, cache=cache)
        dx_l = gs[l - 1] if l > 0 else g        # layer l's dx is layer l-1's incoming gradient
        assert rel_inf(to_np(dx_l), ref_dx) <= 2e-2, ("dx", l)
        for k in ("w1", "w2", "ln1_w", "ln2_w", "b1"):
            e = rel_inf(to_np(grads[l][k]), ref_g[k])
            assert e <= 2e-2, (l, k, e)
    # Stack.step runs the same calls in the same order: the forward is bit-identical; the backward's
    # fp32 reductions (dQ TMA reduce-adds in L2, split-K weight-gradient atomics) sum in an order
    # that varies run to run, so dx may differ in the last bf16 place
    st = D.Stack(jag, m, list(zip(prms, [attn] * n_layers)), X)
    out_s, dx_s, _ = st.step(X, G)
    torch.cuda.synchronize()
    assert torch.equal(out_s, hs[-1])
    assert rel_inf(to_np(dx_s), to_np(g)) <= 1e-2
