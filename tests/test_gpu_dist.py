"""B7 on the GPU (SURVEY §8(e) "Correctness across R"): the CUDA layer's per-shard parameter
gradients, accumulated into one fp32 bucket (uh_layer_bwd accumulate=1, as the data-parallel
step does before its SUM all-reduce), equal the full-batch CUDA gradients to fp32
reassociation tolerance and the oracle to the bf16 bar.  Shards are the LPT assignment of a
skewed jagged batch for R = 2 (the all-reduce itself is covered by tests/test_dist.py)."""
import numpy as np
import pytest
import torch

import oracle as O
from gpu_util import rel_inf, to_dev, to_np
from paper_2602_16986_b200 import dist as D
from paper_2602_16986_b200 import synth
from paper_2602_16986_b200 import uhstu as U

pytestmark = pytest.mark.gpu

NAMES = ("ln1_w", "ln1_b", "w1", "b1", "ln2_w", "ln2_b", "w2", "b2", "pos_bias", "time_bias")


def _layer(cfg, p, pos, ts, t_rows):
    f = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    w = lambda a: torch.from_numpy(a).to("cuda", torch.bfloat16)
    prm = U.Params(f(p["ln1_w"]), f(p["ln1_b"]), w(p["w1"]), f(p["ln2_w"]), f(p["ln2_b"]), w(p["w2"]),
                   f(p["b1"]), f(p["b2"]))
    return prm, U.Attn(cfg.H, cfg.dh, cfg.alpha, float(cfg.N), f(pos), f(ts), f(t_rows))


def test_shard_gradients_accumulate_to_the_full_batch():
    lengths = [1500, 37, 900, 2100, 260, 129, 700, 5]
    cfg = synth.Config("b7", lengths, H=4, dh=128, K1=256, K2=32, N=2200.0, seed=12)
    p = synth.layer_params(cfg.d, cfg.seed)
    x, dout = synth.layer_inputs(cfg)
    pos, ts = synth.rab_tables(cfg)
    t = synth.timestamps(cfg.seed, cfg.lengths)
    m = U.mask(cfg.K1, cfg.K2)
    off = cfg.offsets()
    owner, _ = U.partition_lpt(lengths, 2, m, cfg.d, cfg.H)
    assert set(owner.tolist()) == {0, 1}

    def rows_of(ids):
        return np.concatenate([np.arange(off[i], off[i + 1]) for i in ids])

    # full batch, one call
    prm, attn = _layer(cfg, p, pos, ts, t)
    jag = U.JaggedBatch(off)
    X = to_dev(x, U.BF16)
    _, saved = U.layer_fwd(jag, m, prm, attn, X)
    _, g_full = U.layer_bwd(jag, m, prm, attn, X, saved, to_dev(dout, U.BF16))
    # the two LPT shards, accumulated into one bucket (the rank-local sum the all-reduce adds up)
    bucket = D.GradBucket.for_layer(prm, attn, torch.device("cuda"))
    for r in (0, 1):
        ids = [i for i in range(len(lengths)) if owner[i] == r]
        rows = rows_of(ids)
        prm_r, attn_r = _layer(cfg, p, pos, ts, t[rows])
        jr = U.JaggedBatch.from_lengths([lengths[i] for i in ids])
        Xr = to_dev(x[rows], U.BF16)
        _, sr = U.layer_fwd(jr, m, prm_r, attn_r, Xr)
        U.layer_bwd(jr, m, prm_r, attn_r, Xr, sr, to_dev(dout[rows], U.BF16), grads=bucket.views, accumulate=r > 0)
    torch.cuda.synchronize()
    prm_o = O.LayerParams(**{k: np.asarray(v, np.float64) for k, v in p.items()})
    spec = O.AttnSpec(K1=cfg.K1, K2=cfg.K2, alpha=cfg.alpha, N=float(cfg.N), pos_w=pos, ts_w=ts, timestamps=t)
    _, ref_g = O.layer_backward(dout, off, prm_o, cfg.H, spec, x=x)
    for k in NAMES:
        acc, full = to_np(bucket.views[k]), to_np(g_full[k])
        assert rel_inf(acc, full) <= 1e-5, (k, rel_inf(acc, full))       # fp32 reassociation only
        ok = {"pos_bias": "pos_w", "time_bias": "ts_w"}.get(k, k)
        assert rel_inf(acc, ref_g[ok]) <= 2e-2, (k, rel_inf(acc, ref_g[ok]))
