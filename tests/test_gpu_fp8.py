"""GPU parity of NEXT-2 (FP8 projections) through the C-ABI
(include/uhstu_fp8.h) against the oracle (oracle.quant_rows_e4m3 / gemm_fp8 /
layer_forward_fp8) on identical seeded inputs.

* Weight codes and scales: the oracle quantises by the plain fp64 definition, the kernel
  in fp32 (R19): scales within 1e-6, codes equal except adjacent-grid near-midpoint cases.
* Norm + quant codes: the kernel's LayerNorm is fp32, the oracle's fp64 rounded to
  fp32, so a code may differ only where the value sits within fp32 noise of an E4M3
  rounding midpoint; there it must be the adjacent grid value (R19).  Scales 1e-5.
* FP8 GEMM: fed the oracle's codes, so the only differences are fp32 accumulation
  order and the bf16 output rounding: inf-norm relative error <= 8e-3.
* FP8 layer forward: <= 2e-2 (the north star's bf16 bar).
"""
import numpy as np
import pytest
import torch

import oracle as O
from gpu_util import rel_inf, to_np
from paper_2602_16986_b200 import synth
from paper_2602_16986_b200 import uhstu as U

pytestmark = pytest.mark.gpu


def codes_to_f64(q: torch.Tensor) -> np.ndarray:
    return q.view(torch.float8_e4m3fn).double().cpu().numpy()


def f64_to_codes(v: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(v)).float().to(torch.float8_e4m3fn).view(torch.uint8).cuda()


def bf16(a, seed_shape=None):
    return torch.from_numpy(np.asarray(a, np.float32)).to("cuda", torch.bfloat16)


def bf16_np(t):
    return t.float().cpu().numpy().astype(np.float64)


def check_codes(kq, ks, oq, os_):
    """Row scales within 1e-5; codes equal except rare adjacent-grid near-midpoint cases."""
    assert np.allclose(ks, os_, rtol=1e-5, atol=0)
    diff = kq != oq
    assert diff.mean() < 1e-3, diff.mean()
    if diff.any():
        o, k = oq[diff], kq[diff]
        assert np.all(np.abs(k - o) <= np.maximum(np.abs(o), np.abs(k)) * 2.0 ** -3 + 2.0 ** -9)


@pytest.mark.parametrize("KN", [(512, 2048), (512, 512), (256, 384), (128, 40)])
def test_quant_weight_bit_exact(KN):
    K, N = KN
    r = np.random.default_rng(K + N)
    W = bf16(r.standard_normal((K, N)) * np.exp(r.uniform(-3, 3, (1, N))))
    W[:, 3] = 0
    qt, s = U.quant_weight_fp8(W)
    torch.cuda.synchronize()
    oq, os_ = O.quant_weight_e4m3(bf16_np(W))
    check_codes(codes_to_f64(qt), s.double().cpu().numpy(), oq, os_)
    assert np.allclose(s.double().cpu().numpy(), os_, rtol=1e-6, atol=0)


@pytest.mark.parametrize("T", [1, 7, 1000, 4099])
@pytest.mark.parametrize("d", [512, 256])
def test_ln_and_gated_norm_quant(T, d):
    r = np.random.default_rng(T * d)
    x = bf16(r.standard_normal((T, d)) * 3 + 0.5)
    w = torch.from_numpy(1 + 0.2 * r.standard_normal(d)).float().cuda()
    b = torch.from_numpy(0.1 * r.standard_normal(d)).float().cuda()
    mean = torch.empty(T, device="cuda"); rstd = torch.empty(T, device="cuda")
    q, s = U.ln_fwd_fp8(x, w, b, 1e-6, mean=mean, rstd=rstd)
    torch.cuda.synchronize()
    xh, mu, rs = O.layer_norm(bf16_np(x), w.double().cpu().numpy(), b.double().cpu().numpy(), 1e-6)
    oq, os_ = O.quant_rows_e4m3(xh)
    check_codes(codes_to_f64(q), s.double().cpu().numpy(), oq, os_)
    assert np.allclose(mean.double().cpu().numpy(), mu, rtol=1e-4, atol=1e-5)
    assert np.allclose(rstd.double().cpu().numpy(), rs, rtol=1e-4)
    # gated norm: Y = LN(A) (.) U, U a column block of a wider buffer (row stride 4d)
    A = bf16(r.standard_normal((T, d)))
    UV = bf16(r.standard_normal((T, 4 * d)))
    Ub = UV[:, :d]
    q2, s2 = U.gated_norm_fwd_fp8(A, Ub, w, b, 1e-6)
    torch.cuda.synchronize()
    ah, _, _ = O.layer_norm(bf16_np(A), w.double().cpu().numpy(), b.double().cpu().numpy(), 1e-6)
    oq2, os2 = O.quant_rows_e4m3(ah * bf16_np(Ub))
    check_codes(codes_to_f64(q2), s2.double().cpu().numpy(), oq2, os2)


def test_all_zero_row_gets_unit_scale():
    x = torch.zeros(3, 256, dtype=torch.bfloat16, device="cuda")
    w = torch.zeros(256, device="cuda"); b = torch.zeros(256, device="cuda")
    q, s = U.ln_fwd_fp8(x, w, b)
    torch.cuda.synchronize()
    assert torch.all(q == 0) and torch.all(s == 1)


# M ragged (several tiles + tail; 37965 rows: every CTA walks several tiles), N in 256 and 128 tiles
@pytest.mark.parametrize("MNK", [(200, 512, 256), (1000, 2048, 512), (37965, 512, 128), (300, 384, 512)])
@pytest.mark.parametrize("epi", [0, 1])
def test_gemm_fp8_against_oracle(MNK, epi):
    M, N, K = MNK
    r = np.random.default_rng(M + N + K + epi)
    a = r.standard_normal((M, K)) * np.exp(r.uniform(-2, 2, (M, 1)))
    w = r.standard_normal((K, N)) / np.sqrt(K)
    qa, sa = O.quant_rows_e4m3(a)
    qb, sb = O.quant_weight_e4m3(w)
    bias = r.standard_normal(N) * 0.3
    resid = bf16(r.standard_normal((M, N))) if epi == 0 else None
    out = U.gemm_fp8(f64_to_codes(qa), torch.from_numpy(sa).float().cuda(), f64_to_codes(qb),
                     torch.from_numpy(sb).float().cuda(), epi, bias=torch.from_numpy(bias).float().cuda(),
                     resid=resid)
    torch.cuda.synchronize()
    h = O.gemm_fp8(qa, sa, qb, sb) + bias[None, :]
    ref = h + bf16_np(resid) if epi == 0 else O.silu(h)
    assert rel_inf(to_np(out), ref) < 8e-3


def test_gemm_fp8_rejects_bad_shapes():
    q = torch.zeros(128, 96, dtype=torch.uint8, device="cuda")
    s = torch.ones(128, device="cuda")
    with pytest.raises(U.UhError):
        U.gemm_fp8(q, s, q, s)          # K = 96 is not a multiple of 128


@pytest.mark.parametrize("name", ["tiny128", "mid512"])
def test_layer_fwd_fp8_against_oracle(name):
    # mid512: the cfg3 widths (4 heads x 128, rab) on ragged lengths spanning several 128-row tiles
    cfg = synth.config(name) if name != "mid512" else \
        synth.Config("mid512", [300, 1025, 77], H=4, dh=128, K1=256, K2=16, N=2048, seed=5, pos_len=128)
    p = synth.layer_params(cfg.d, cfg.seed)
    x, _ = synth.layer_inputs(cfg)
    pos, ts = synth.rab_tables(cfg)
    t = synth.timestamps(cfg.seed, cfg.lengths)
    f = lambda a: torch.from_numpy(a).cuda()
    b = lambda a: torch.from_numpy(a).to("cuda", torch.bfloat16)
    prm = U.Params(f(p["ln1_w"]), f(p["ln1_b"]), b(p["w1"]), f(p["ln2_w"]), f(p["ln2_b"]), b(p["w2"]),
                   f(p["b1"]), f(p["b2"]))
    attn = U.Attn(cfg.H, cfg.dh, 1.0, float(cfg.N), f(pos), f(ts), f(t))
    jag = U.JaggedBatch(cfg.offsets())
    m = U.mask(cfg.K1, cfg.K2)
    X = b(x)
    qw = U.quant_layer_weights(prm)
    out, saved = U.layer_fwd_fp8(jag, m, prm, attn, X, qw, save=True)
    torch.cuda.synchronize()
    # the oracle sees the same bf16 weights and input the GPU path does
    po = {k: np.asarray(v, np.float64) for k, v in p.items()}
    po["w1"] = bf16_np(prm.w1); po["w2"] = bf16_np(prm.w2)
    prm_o = O.LayerParams(**po)
    spec = O.AttnSpec(K1=cfg.K1, K2=cfg.K2, alpha=1.0, N=cfg.N, pos_w=pos, ts_w=ts, timestamps=t)
    r_out, cache = O.layer_forward_fp8(bf16_np(X), cfg.offsets(), prm_o, cfg.H, spec)
    assert rel_inf(to_np(out), r_out) < 2e-2
    assert rel_inf(to_np(saved.attn), cache["A"]) < 2e-2
    # and it is the FP8 path: the bf16 layer differs from it by more than rounding noise
    r_bf, _ = O.layer_forward(bf16_np(X), cfg.offsets(), prm_o, cfg.H, spec)
    assert np.max(np.abs(r_out - r_bf)) > 0
