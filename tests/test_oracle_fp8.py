"""Pins for the oracle's FP8 projections (NEXT-2), CPU only.

The E4M3 rounding is pinned to the format's definition (the grid enumerated from
its bit fields) and to torch's float8_e4m3fn cast (a library routine); the
row-wise quantisation to its invariants and to a brute-force nearest-grid search;
the scaled GEMM to exact integer-grid arithmetic; the FP8 layer to the rigorous
worst-case error bound of the two quantisations.
"""
import numpy as np
import torch

import oracle as O
from paper_2602_16986_b200 import synth


def e4m3_grid():
    """All finite non-negative E4M3FN values from the bit fields (bias 7, no inf,
    exponent 15 / mantissa 7 is NaN)."""
    vals = []
    for e in range(16):
        for m in range(8):
            if e == 15 and m == 7:
                continue
            vals.append(m / 8 * 2.0 ** -6 if e == 0 else (1 + m / 8) * 2.0 ** (e - 7))
    return np.array(sorted(vals))


def test_e4m3_grid_fixed_points_and_extremes():
    g = e4m3_grid()
    assert len(g) == 127 and g[-1] == 448.0 and g[1] == 2.0 ** -9
    assert np.array_equal(O.e4m3_round(g), g)
    assert np.array_equal(O.e4m3_round(-g), -g)
    # saturation (satfinite) and the smallest values
    assert np.array_equal(O.e4m3_round([448.0, 460.0, 1e6, -1e6]), [448.0, 448.0, 448.0, -448.0])
    assert O.e4m3_round(2.0 ** -10) == 0.0                 # tie between 0 and 2^-9 -> even (0)
    assert O.e4m3_round(1.5 * 2.0 ** -9) == 2.0 ** -8      # tie between 1 and 2 (x 2^-9) -> even (2)
    assert O.e4m3_round(0.76 * 2.0 ** -9) == 2.0 ** -9


def test_e4m3_midpoints_tie_to_even_mantissa():
    g = e4m3_grid()
    mids = (g[:-1] + g[1:]) / 2
    r = O.e4m3_round(mids)
    for lo, hi, v in zip(g[:-1], g[1:], r):
        # even = the neighbour whose last mantissa bit is 0 (code index parity on the sorted grid)
        i_lo = int(np.searchsorted(g, lo))
        assert v == (lo if i_lo % 2 == 0 else hi)


def test_e4m3_matches_torch_float8_cast():
    r = np.random.default_rng(0)
    v = np.concatenate([r.standard_normal(50000) * 60, r.standard_normal(20000) * 2.0 ** -7,
                        r.uniform(-448, 448, 20000)]).astype(np.float32)
    ours = O.e4m3_round(v.astype(np.float64))
    ref = torch.from_numpy(v).to(torch.float8_e4m3fn).double().numpy()
    assert np.array_equal(ours, ref)


def test_quant_rows_invariants_and_brute_force():
    r = np.random.default_rng(1)
    x = r.standard_normal((40, 96)) * np.exp(r.uniform(-6, 6, (40, 1)))
    x[3] = 0.0
    q, s = O.quant_rows_e4m3(x)
    g = e4m3_grid()
    gs = np.concatenate([-g[::-1], g])
    nz = np.arange(40) != 3
    assert np.all(np.abs(q[nz]).max(axis=1) == 448.0)      # the row maximum maps to the top code
    assert np.all(q[3] == 0) and s[3] == 1.0
    # every code is the nearest grid value to x / s (brute force over the grid)
    assert np.allclose(s[nz], np.abs(x[nz]).max(axis=1) / 448.0, rtol=1e-15, atol=0)
    t = x[nz] / s[nz, None]
    dist = np.abs(t[..., None] - gs)
    near = gs[np.argmin(dist, axis=-1)]
    tie = np.sort(dist, axis=-1)[..., 1] - np.sort(dist, axis=-1)[..., 0] < 1e-12 * np.maximum(1, np.abs(t))
    assert np.array_equal(near[~tie], q[nz][~tie])          # nearest grid value, decided in fp64
    # half-ulp reconstruction bound: |q s - x| <= 2^-4 |x| + 2^-10 s
    err = np.abs(q * s[:, None] - x)
    assert np.all(err <= (2.0 ** -4 * np.abs(x) + 2.0 ** -10 * s[:, None]) * (1 + 1e-12))
    # weight quantisation is per output column: W[:, n] ~= qT[n] s[n]
    w = r.standard_normal((64, 32))
    qT, sw = O.quant_weight_e4m3(w)
    assert qT.shape == (32, 64) and sw.shape == (32,)
    assert np.all(np.abs(qT).max(axis=1) == 448.0)
    assert np.all(np.abs(qT * sw[:, None] - w.T) <= 2.0 ** -4 * np.abs(w.T) + 2.0 ** -10 * sw[:, None] + 1e-12)


def test_quant_rows_hand_example():
    # row [1, -2, 0.3]: s = 2/448; x/s = [224, -448, 67.2] -> codes [224, -448, 64]
    # (E4M3 spacing in [64, 128) is 8, so 67.2 rounds to 64); all-zero row: s = 1
    q, s = O.quant_rows_e4m3(np.array([[1.0, -2.0, 0.3], [0.0, 0.0, 0.0]]))
    assert np.allclose(s, [2.0 / 448.0, 1.0], rtol=1e-15)
    assert np.array_equal(q, [[224.0, -448.0, 64.0], [0.0, 0.0, 0.0]])


def test_gemm_fp8_exact_on_the_grid():
    # hand example: D = diag(sa) (qa qb^T) diag(sb)
    qa = np.array([[1.0, 2.0], [3.0, -4.0]])
    qbT = np.array([[0.5, 1.0], [2.0, 0.0], [-1.0, 448.0]])
    d = O.gemm_fp8(qa, [2.0, 0.25], qbT, [1.0, 4.0, 0.5])
    assert np.array_equal(d, [[5.0, 16.0, 895.0], [-0.625, 6.0, -224.375]])
    # random grid codes with power-of-two scales: exact integer-grid arithmetic
    r = np.random.default_rng(2)
    g = e4m3_grid()
    A = r.choice(np.concatenate([-g, g]), (17, 64))
    B = r.choice(np.concatenate([-g, g]), (24, 64))
    sa = 2.0 ** r.integers(-8, 8, 17)
    sb = 2.0 ** r.integers(-8, 8, 24)
    ref = (A * sa[:, None]) @ (B * sb[:, None]).T
    assert np.array_equal(O.gemm_fp8(A, sa, B, sb), ref)


def _bound(a, sa, bT, sb):
    """Worst case |FP8GEMM - exact| for A [M,K] (row scales sa) and B^T [N,K] (row scales sb)."""
    ea = 2.0 ** -4 * np.abs(a) + 2.0 ** -10 * sa[:, None]
    eb = 2.0 ** -4 * np.abs(bT) + 2.0 ** -10 * sb[:, None]
    return (ea @ (np.abs(bT) + eb).T + np.abs(a) @ eb.T) * (1 + 1e-5)


def test_layer_forward_fp8_within_the_quantisation_bound():
    cfg = synth.Config("t", [5, 37, 64], H=2, dh=32, K1=8, K2=2, N=64.0, seed=3)
    d = cfg.H * cfg.dh
    p = synth.layer_params(d, cfg.seed)
    prm = O.LayerParams(**{k_: np.asarray(v_, np.float64) for k_, v_ in p.items()})
    x = np.random.default_rng(3).standard_normal((cfg.T, d))
    spec = O.AttnSpec(K1=cfg.K1, K2=cfg.K2, alpha=1.0, N=cfg.N)
    out8, c8 = O.layer_forward_fp8(x, cfg.offsets(), prm, cfg.H, spec)
    out, c = O.layer_forward(x, cfg.offsets(), prm, cfg.H, spec)
    # f1: the FP8 GEMM + b1 is within the bound of the exact x^ W1 + b1 (same x^)
    assert np.array_equal(c8["xh"], c["xh"])
    _, sw1 = O.quant_weight_e4m3(prm.w1)
    b1 = _bound(c["xh"], c8["sx"], prm.w1.T, sw1)
    assert np.all(np.abs(c8["h"] - c["h"]) <= b1)
    assert np.max(np.abs(c8["h"] - c["h"])) > 0               # it is quantised
    # f2: out - x - b2 against the exact Y8 W2 of the FP8 path's own Y
    _, sw2 = O.quant_weight_e4m3(prm.w2)
    f2_exact = c8["Y"] @ prm.w2
    b2 = _bound(c8["Y"], c8["sy"], prm.w2.T, sw2)
    assert np.all(np.abs(out8 - x - prm.b2[None, :] - f2_exact) <= b2 + 1e-12)
    # and the whole layer stays within one E4M3 rounding step (2^-4 relative, R17) of the
    # fp64 layer (infinity-norm relative, R15)
    assert np.max(np.abs(out8 - out)) / np.max(np.abs(out)) < 2.0 ** -4
