"""GPU parity: the CUDA path (through the C-ABI) against the fp64 oracle, element by
element, on identical seeded inputs.  Bars (BASELINE.json north star): per-tensor
infinity-norm relative error <= 2e-2 for bf16 I/O with fp32 accumulation, <= 1e-4
for the fp32 verification build."""
import numpy as np
import pytest
import torch

import oracle as O
from gpu_util import AttnCase, rel_inf, to_dev, to_np, tdt
from paper_2602_16986_b200 import synth
from paper_2602_16986_b200 import uhstu as U

pytestmark = pytest.mark.gpu

TOL = {U.BF16: 2e-2, U.F32: 1e-4}

# lengths that straddle tile boundaries (SURVEY §8(c) parity matrix)
RAGGED = [0, 1, 2, 17, 63, 64, 65, 127, 128, 129, 255, 256, 257]


# ----------------------------------------------------------------------------- GEMM (test hook)
@pytest.mark.parametrize("a_mn,b_mn", [(False, False), (False, True), (True, True)])
# (37965, 512, 128): 298 CTA-pair tiles over 74 pairs with a ragged last pair tile -- every CTA
# walks several tiles (both TMEM accumulators, barrier phase flips)
@pytest.mark.parametrize("MNK", [(256, 512, 128), (296, 256, 192), (128, 2048, 512), (768, 512, 1024),
                                 (37965, 512, 128)])
@pytest.mark.parametrize("pair", [0, 2])   # 2: CTA-pair (cta_group::2) tiles where eligible
def test_gemm_bf16_majors(a_mn, b_mn, MNK, pair):
    M, N, K = MNK
    if a_mn and M % 8:
        pytest.skip("MN-major A is stored [K][M]: its row stride M must be a multiple of 8")
    g = torch.Generator().manual_seed(0)
    A = torch.randn(M, K, generator=g).bfloat16()
    B = torch.randn(K, N, generator=g).bfloat16()
    ref = (A.double() @ B.double())
    Ad = (A.t().contiguous() if a_mn else A).cuda()
    Bd = (B.contiguous() if b_mn else B.t().contiguous()).cuda()
    if a_mn:
        out, _ = U.test_gemm(Ad, Bd, True, b_mn, 2, M, N, K, cta_pair=pair)
    else:
        out, _ = U.test_gemm(Ad, Bd, False, b_mn, 0, M, N, K, cta_pair=pair)
    torch.cuda.synchronize()
    assert rel_inf(to_np(out), ref.numpy()) < (1e-5 if a_mn else 8e-3)


@pytest.mark.parametrize("b_mn", [True, False])
@pytest.mark.parametrize("M", [200, 20000])
@pytest.mark.parametrize("pair", [0, 2])
def test_gemm_bf16_silu_and_residual_epilogues(b_mn, M, pair):
    N, K = 512, 256
    g = torch.Generator().manual_seed(1)
    A = torch.randn(M, K, generator=g).bfloat16()
    B = (torch.randn(K, N, generator=g) / 16).bfloat16()
    bias = torch.randn(N, generator=g)
    R = torch.randn(M, N, generator=g).bfloat16()
    h = A.double() @ B.double() + bias.double()
    s = torch.sigmoid(h)
    out0 = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    out1 = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    U.test_gemm(A.cuda(), (B if b_mn else B.t()).contiguous().cuda(), False, b_mn, 1, M, N, K, bias=bias.cuda(),
                out0=out0, out1=out1, cta_pair=pair)
    torch.cuda.synchronize()
    assert rel_inf(to_np(out0), (h * s).numpy()) < 8e-3
    assert rel_inf(to_np(out1), (s * (1 + h * (1 - s))).numpy()) < 8e-3
    out, _ = U.test_gemm(A.cuda(), (B if b_mn else B.t()).contiguous().cuda(), False, b_mn, 0, M, N, K,
                         bias=bias.cuda(), resid=R.cuda(), cta_pair=pair)
    torch.cuda.synchronize()
    assert rel_inf(to_np(out), (h + R.double()).numpy()) < 8e-3


# ----------------------------------------------------------------------------- attention forward
def run_fwd(case: AttnCase, dtype, fused=True):
    jag = case.jag()
    if fused:
        _, q, k, v = case.fused_qkv(dtype)
    else:
        q, k, v = to_dev(case.q, dtype), to_dev(case.k, dtype), to_dev(case.v, dtype)
    A = U.attn_fwd(jag, case.mask(), case.desc(), q, k, v)
    torch.cuda.synchronize()
    return to_np(A)


def oracle_fwd(case: AttnCase):
    c = case.cfg
    return O.attention_forward(c.offsets(), c.H, c.dh, case.q, case.k, case.v, case.spec())


def test_attn_fwd_f32_tiny():
    cfg = synth.config("tiny")
    case = AttnCase(cfg.lengths, H=cfg.H, dh=cfg.dh, K1=cfg.K1, K2=cfg.K2, N=cfg.N, seed=cfg.seed)
    assert rel_inf(run_fwd(case, U.F32, fused=False), oracle_fwd(case)) <= TOL[U.F32]


@pytest.mark.parametrize("dtype", [U.BF16, U.F32])
def test_attn_fwd_tiny128(dtype):
    case = AttnCase([17, 40, 64], H=2, dh=128, K1=16, K2=2, N=64)
    assert rel_inf(run_fwd(case, dtype), oracle_fwd(case)) <= TOL[dtype]


@pytest.mark.parametrize("K1,K2", [(16, 2), (0, 0), (1, 0), (127, 129), (128, 1), (129, 300), (synth.WINDOW_FULL, 0)])
@pytest.mark.parametrize("dtype", [U.BF16, U.F32])
def test_attn_fwd_ragged_matrix(K1, K2, dtype):
    case = AttnCase(RAGGED + [K1 % 700 + 1, 300], H=2, dh=128, K1=K1, K2=K2, N=300.0, P=40, seed=5)
    assert rel_inf(run_fwd(case, dtype), oracle_fwd(case)) <= TOL[dtype]


def test_attn_fwd_no_rab_alpha():
    case = AttnCase([130, 900, 7], H=4, dh=128, K1=200, K2=20, N=900.0, rab=False, alpha=0.37, seed=9)
    assert rel_inf(run_fwd(case, U.BF16), oracle_fwd(case)) <= TOL[U.BF16]


def test_attn_fwd_cfg2_like_full_causal():
    lengths = synth.lengths_uniform(2, 6, 1024, 2048)
    case = AttnCase(lengths, H=4, dh=128, K1=synth.WINDOW_FULL, K2=0, N=4096.0, seed=2, P=128)
    assert rel_inf(run_fwd(case, U.BF16), oracle_fwd(case)) <= TOL[U.BF16]


# ----------------------------------------------------------------------------- attention backward
def run_bwd(case: AttnCase, dtype):
    jag = case.jag()
    _, q, k, v = case.fused_qkv(dtype)
    dA = to_dev(case.dA, dtype)
    dq, dk, dv, dpos, dts = U.attn_bwd(jag, case.mask(), case.desc(), q, k, v, dA)
    torch.cuda.synchronize()
    return [to_np(x) if x is not None else None for x in (dq, dk, dv, dpos, dts)]


def oracle_bwd(case: AttnCase):
    c = case.cfg
    return O.attention_backward(c.offsets(), c.H, c.dh, case.q, case.k, case.v, case.dA, case.spec(),
                                return_abs=True)


def check_bwd(case, dtype):
    got = run_bwd(case, dtype)
    ref = oracle_bwd(case)
    for n, g, r in zip(["dQ", "dK", "dV"], got[:3], ref[:3]):
        e = rel_inf(g, r)
        assert e <= TOL[dtype], (n, e)
    # d pos_bias / d time_bias: sums of ds of both signs over many pairs per entry; the bar
    # applies per entry to the summation-error scale sum |ds| (R15b)
    for n, g, r, ra in zip(["dpos", "dts"], got[3:5], ref[3:5], ref[5:7]):
        if r is None:
            continue
        err = np.abs(np.asarray(g, np.float64) - r)
        assert np.all(err <= TOL[dtype] * ra + 1e-12), (n, float(np.max(err / (ra + 1e-30))))


def test_attn_bwd_f32_tiny():
    cfg = synth.config("tiny")
    case = AttnCase(cfg.lengths, H=cfg.H, dh=cfg.dh, K1=cfg.K1, K2=cfg.K2, N=cfg.N, seed=cfg.seed)
    check_bwd(case, U.F32)


# SURVEY §8(c) parity matrix for the backward (and the forward on the same cases): windows K1
# in {0, 1, 15, 16, 127, 128, 129, 1024, full}, global prefixes K2 in {0, 1, 2, 127, 128, 129,
# > K1, >= L} (each K1 with a rotating selection of four), and one jagged batch mixing the
# ragged tile-boundary lengths with {K1, K1+1, K1+2, K1+K2, K1+K2+1, K1+BM, K1+BM+1} (BM = 128).
# The position table alternates between a short P (most offsets clamp to P-1) and P >= every
# length (every offset its own entry).
K1S = [0, 1, 15, 16, 127, 128, 129, 1024, synth.WINDOW_FULL]
K2S = [0, 1, 2, 127, 128, 129, "gtK1", "geL"]
BWD_CASES = []
for _i, _k1 in enumerate(K1S):
    for _j in range(4):
        _k2 = K2S[(2 * _i + _j) % len(K2S)]
        BWD_CASES.append((_k1, _k2, 40 if (_i + _j) % 2 else 5000))


def matrix_case(K1, K2, P, seed):
    fin = K1 < synth.WINDOW_FULL
    if K2 == "gtK1":
        K2 = (K1 + 1) if fin else 300
    if K2 == "geL":
        K2 = 4000
    extra = [K1, K1 + 1, K1 + 2, K1 + K2, K1 + K2 + 1, K1 + 128, K1 + 129] if fin else [700, 1300]
    lengths = RAGGED + sorted({min(L, 1400) for L in extra if L > 0})
    return AttnCase(lengths, H=2, dh=128, K1=K1, K2=K2, N=1400.0, P=P, seed=6 + K1 % 97 + 3 * (K2 % 13))


@pytest.mark.parametrize("K1,K2,P", BWD_CASES)
@pytest.mark.parametrize("dtype", [U.BF16, U.F32])
def test_attn_bwd_ragged_matrix(K1, K2, P, dtype):
    case = matrix_case(K1, K2, P, 6)
    check_bwd(case, dtype)
    assert rel_inf(run_fwd(case, dtype), oracle_fwd(case)) <= TOL[dtype]


@pytest.mark.parametrize("K1,K2", [(1024, 128), (synth.WINDOW_FULL, 0)])
def test_attn_position_table_longer_than_sequences(K1, K2):
    """P = 16384 (the cfg3 reading: one entry per offset up to the max length) on sequences of
    several hundred tiles: every offset reads its own entry; fwd and bwd against the oracle."""
    case = AttnCase([3000, 1, 2200, 129], H=2, dh=128, K1=K1, K2=K2, N=16384.0, P=16384, seed=11)
    assert rel_inf(run_fwd(case, U.BF16), oracle_fwd(case)) <= TOL[U.BF16]
    check_bwd(case, U.BF16)


# ----------------------------------------------------------------------------- layer
def test_attn_row_strides_off_32_bytes():
    """Output / gradient row strides that are 16- but not 32-byte multiples (width + 8 elements):
    the per-thread O, dV, dK rows then take the 16-byte store path instead of the 32-byte one."""
    case = AttnCase([70, 300, 129], H=2, dh=128, K1=64, K2=8, N=300.0, P=400, seed=3)
    jag = case.jag()
    w = case.cfg.H * case.cfg.dh
    _, q, k, v = case.fused_qkv(U.BF16)
    out = torch.empty(q.shape[0], w + 8, dtype=torch.bfloat16, device="cuda")[:, :w]
    A = U.attn_fwd(jag, case.mask(), case.desc(), q, k, v, out=out)
    g = torch.empty(q.shape[0], 3 * w + 8, dtype=torch.bfloat16, device="cuda")
    dq, dk, dv = g[:, :w], g[:, w:2 * w], g[:, 2 * w:3 * w]
    U.attn_bwd(jag, case.mask(), case.desc(), q, k, v, to_dev(case.dA, U.BF16), dq=dq, dk=dk, dv=dv)
    torch.cuda.synchronize()
    assert out.stride(0) * 2 % 32 and g.stride(0) * 2 % 32
    assert rel_inf(to_np(A), oracle_fwd(case)) <= TOL[U.BF16]
    ref = oracle_bwd(case)
    for n, got, r in zip(("dQ", "dK", "dV"), (dq, dk, dv), ref[:3]):
        e = rel_inf(to_np(got), r)
        assert e <= TOL[U.BF16], (n, e)


def layer_case(cfg, dtype, biases=True):
    p = synth.layer_params(cfg.d, cfg.seed, biases=biases)
    x, dout = synth.layer_inputs(cfg)
    pos, ts = synth.rab_tables(cfg)
    t = synth.timestamps(cfg.seed, cfg.lengths)
    return p, x, dout, pos, ts, t


def gpu_params(p, dtype):
    f = lambda a: torch.from_numpy(a).cuda()
    w = lambda a: torch.from_numpy(a).to("cuda", tdt(dtype))
    return U.Params(f(p["ln1_w"]), f(p["ln1_b"]), w(p["w1"]), f(p["ln2_w"]), f(p["ln2_b"]), w(p["w2"]),
                    f(p["b1"]) if "b1" in p else None, f(p["b2"]) if "b2" in p else None)


def oracle_layer(cfg, p, x, dout, pos, ts, t):
    prm = O.LayerParams(**{k: np.asarray(v, np.float64) for k, v in p.items()})
    spec = O.AttnSpec(K1=O.FULL if cfg.K1 >= synth.WINDOW_FULL else cfg.K1, K2=cfg.K2, alpha=cfg.alpha, N=cfg.N,
                      pos_w=pos, ts_w=ts, timestamps=t)
    out, cache = O.layer_forward(x, cfg.offsets(), prm, cfg.H, spec)
    dx, g = O.layer_backward(dout, cfg.offsets(), prm, cfg.H, spec, cache=cache)
    return out, dx, g


def run_layer(cfg, dtype, p, x, dout, pos, ts, t):
    jag = U.JaggedBatch(cfg.offsets())
    prm = gpu_params(p, dtype)
    attn = U.Attn(cfg.H, cfg.dh, cfg.alpha, float(cfg.N), torch.from_numpy(pos).cuda(), torch.from_numpy(ts).cuda(),
                  torch.from_numpy(t).cuda())
    m = U.mask(cfg.K1, cfg.K2)
    X = to_dev(x, dtype)
    out, saved = U.layer_fwd(jag, m, prm, attn, X)
    dx, grads = U.layer_bwd(jag, m, prm, attn, X, saved, to_dev(dout, dtype))
    torch.cuda.synchronize()
    return to_np(out), to_np(dx), {k: to_np(v) for k, v in grads.items() if v is not None}, saved


@pytest.mark.parametrize("name,dtype", [("tiny", U.F32), ("tiny128", U.F32), ("tiny128", U.BF16)])
def test_layer_fwd_bwd(name, dtype):
    cfg = synth.config(name)
    p, x, dout, pos, ts, t = layer_case(cfg, dtype)
    out, dx, g, _ = run_layer(cfg, dtype, p, x, dout, pos, ts, t)
    r_out, r_dx, r_g = oracle_layer(cfg, p, x, dout, pos, ts, t)
    assert rel_inf(out, r_out) <= TOL[dtype]
    assert rel_inf(dx, r_dx) <= TOL[dtype]
    for k in ("ln1_w", "ln1_b", "w1", "b1", "ln2_w", "ln2_b", "w2", "b2", "pos_bias", "time_bias"):
        ok = {"pos_bias": "pos_w", "time_bias": "ts_w"}.get(k, k)
        assert rel_inf(g[k], r_g[ok]) <= TOL[dtype], (k, rel_inf(g[k], r_g[ok]))


# ----------------------------------------------------------------------------- jagged ops
def test_jagged_gather_slice_padded():
    lengths = [5, 0, 17, 64, 3]
    jag = U.JaggedBatch.from_lengths(lengths)
    x = torch.arange(sum(lengths) * 8, dtype=torch.float32, device="cuda").reshape(-1, 8)
    xn = to_np(x)
    off = jag.host
    y, j2 = U.jagged_gather(jag, [3, 0, 2], x)
    ref = np.concatenate([xn[off[3]:off[4]], xn[off[0]:off[1]], xn[off[2]:off[3]]])
    assert np.array_equal(to_np(y), ref) and list(j2.lengths) == [64, 5, 17]
    y, j3 = U.jagged_slice_latest(jag, 4, x)
    ref = np.concatenate([xn[off[b + 1] - min(4, L):off[b + 1]] for b, L in enumerate(lengths)])
    assert np.array_equal(to_np(y), ref) and list(j3.lengths) == [4, 0, 4, 4, 3]
    pad = U.jagged_to_padded(jag, x, 64)
    back = U.padded_to_jagged(jag, pad)
    assert np.array_equal(to_np(back), xn)
    assert float(pad[0, 5:].abs().sum()) == 0.0


def test_jagged_gather_odd_8byte_stride():
    """16-byte rows read from a view whose row stride is an odd multiple of 8 bytes (width 8 bf16,
    ld 12): every odd row starts 8 bytes off a 16-byte boundary, so the copy must take the
    8-byte path (a 16-byte vector load there faults)."""
    lengths = [3, 6, 1, 9]
    jag = U.JaggedBatch.from_lengths(lengths)
    base = torch.arange(sum(lengths) * 12, dtype=torch.float32).reshape(-1, 12).to("cuda", torch.bfloat16)
    x = base[:, :8]
    assert x.stride(0) == 12
    y, j2 = U.jagged_gather(jag, [3, 1, 0], x)
    y2, _ = U.jagged_slice_latest(jag, 2, x)
    torch.cuda.synchronize()
    xn, off = to_np(x), jag.host
    assert np.array_equal(to_np(y), np.concatenate([xn[off[3]:off[4]], xn[off[1]:off[2]], xn[off[0]:off[1]]]))
    assert np.array_equal(to_np(y2), np.concatenate([xn[off[b + 1] - min(2, L):off[b + 1]]
                                                     for b, L in enumerate(lengths)]))
