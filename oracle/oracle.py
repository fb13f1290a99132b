"""ORACLE — test infrastructure only.

Plain, slow, obviously-correct fp64 CPU implementation of the ULTRA-HSTU layer
(arXiv 2602.16986) hot path.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import it.  It shares
no code with the CUDA path (``paper_2602_16986_b200``) and the CUDA path never
imports it.  The seeded input generators live in ``paper_2602_16986_b200/synth.py``
(no method arithmetic there) and are the only thing both sides use.

Every function cites the passage it follows; PAPER.md = /root/reference/PAPER.md,
``P:n`` = its line n; ``R<k>`` = reading k in DESIGN.md §3 (where the paper is
silent or garbled).

* layer_forward  — Eqs. 1-5 in Listing 1's order:
      x^ = Norm(x); U,V,Q,K = SiLU(x^ W1 + b1); A = attention(Q,K,V);
      Y = Norm(A) (.) U; out = Y W2 + b2 + x.
* layer_backward — the exact chain rule of layer_forward; Listing 1
  fixes the set of gradients returned (dx, d_norm_w, d_linear_w_1,
  d_gated_norm_w, d_linear_w_2) and ``dx += dout``.
* attention_forward / attention_backward — the C pair loops in attn_oracle.c
  (Eq. 3; SLA mask P:140-146).
* layer_forward_fp8 / quant_rows_e4m3 / gemm_fp8 — NEXT-2, both projections in
  row-wise scaled E4M3 (readings R17-R20).
* partition_lpt — the token-balanced partitioner: LPT on the cost model of
  DESIGN.md §6; the load notion follows LBSL's
  "load of a rank ... sum n_u^gamma".

Matmuls are numpy (a library primitive used as one step); nothing is blocked,
fused or reordered beyond the equations.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "attn_oracle.c")
_LIB_PATH = os.path.join(_HERE, "build", "libattn_oracle.so")
_lib = None

FULL = -1  # K1 < 0 selects full causal in the oracle


def build(force: bool = False) -> str:
    """Compile attn_oracle.c (plain C, -O2, OpenMP) into oracle/build/."""
    os.makedirs(os.path.dirname(_LIB_PATH), exist_ok=True)
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        tmp = _LIB_PATH + ".tmp%d" % os.getpid()
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11",
                               "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        i32p = ctypes.POINTER(ctypes.c_int32)
        i64p = ctypes.POINTER(ctypes.c_int64)
        dp = ctypes.POINTER(ctypes.c_double)
        I64, D = ctypes.c_int64, ctypes.c_double
        _lib.orc_mask_allows.argtypes = [I64, I64, I64, I64]
        _lib.orc_mask_allows.restype = ctypes.c_int
        _lib.orc_mask_nnz.argtypes = [I64, I64, I64]
        _lib.orc_mask_nnz.restype = I64
        _lib.orc_attn_fwd.argtypes = [ctypes.c_int, i32p, ctypes.c_int, ctypes.c_int,
                                      dp, dp, dp, I64, I64, I64, D, D,
                                      dp, I64, dp, I64, i64p, dp, I64, i64p]
        _lib.orc_attn_fwd.restype = None
        _lib.orc_attn_bwd.argtypes = [ctypes.c_int, i32p, ctypes.c_int, ctypes.c_int,
                                      dp, dp, dp, I64, dp, I64, I64, I64, D, D,
                                      dp, I64, dp, I64, i64p,
                                      dp, dp, dp, I64, dp, dp, dp, dp, i64p]
        _lib.orc_attn_bwd.restype = None
        _lib.orc_num_threads.restype = ctypes.c_int
    return _lib


def num_threads() -> int:
    return int(_load().orc_num_threads())


def _ptr(a, ctype):
    if a is None:
        return None
    return a.ctypes.data_as(ctypes.POINTER(ctype))


def _f64(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float64)


# ----------------------------------------------------------------------------
# mask (readings R1-R4)
# ----------------------------------------------------------------------------
def mask_allows(q: int, k: int, K1: int, K2: int) -> bool:
    return bool(_load().orc_mask_allows(q, k, K1, K2))


def mask_nnz(L: int, K1: int, K2: int) -> int:
    """Allowed pairs of a length-L sequence, counted by enumeration."""
    return int(_load().orc_mask_nnz(L, K1, K2))


# ----------------------------------------------------------------------------
# attention (Eq. 3) — C pair loops
# ----------------------------------------------------------------------------
@dataclass
class AttnSpec:
    """Mask + normalisation + rab of one layer (R1-R7)."""
    K1: int = FULL              # window (inclusive); FULL (<0) = causal
    K2: int = 0                 # global prefix tokens
    alpha: float = 1.0          # score scale (R6)
    N: float = 1.0              # silu(.)/N normaliser (R5)
    pos_w: Optional[np.ndarray] = None   # [P]  (R7)
    ts_w: Optional[np.ndarray] = None    # [NB] (R7)
    timestamps: Optional[np.ndarray] = None  # int64 [T]


def attention_forward(offsets, H, dh, q, k, v, spec: AttnSpec, return_work=False):
    """A[r, h*dh:(h+1)*dh] for the jagged batch.  q,k,v: [T, >=H*dh] fp64."""
    lib = _load()
    offsets = np.ascontiguousarray(offsets, dtype=np.int32)
    B = len(offsets) - 1
    q, k, v = _f64(q), _f64(k), _f64(v)
    T = int(offsets[-1])
    ld = q.shape[1]
    assert k.shape[1] == ld and v.shape[1] == ld
    A = np.zeros((T, H * dh), dtype=np.float64)
    pos = _f64(spec.pos_w)
    ts = _f64(spec.ts_w)
    t = None
    if ts is not None:
        t = np.ascontiguousarray(spec.timestamps, dtype=np.int64)
    work = ctypes.c_int64(0)
    lib.orc_attn_fwd(B, _ptr(offsets, ctypes.c_int32), H, dh,
                     _ptr(q, ctypes.c_double), _ptr(k, ctypes.c_double), _ptr(v, ctypes.c_double), ld,
                     spec.K1, spec.K2, float(spec.alpha), float(spec.N),
                     _ptr(pos, ctypes.c_double), 0 if pos is None else len(pos),
                     _ptr(ts, ctypes.c_double), 0 if ts is None else len(ts),
                     _ptr(t, ctypes.c_int64), _ptr(A, ctypes.c_double), H * dh, ctypes.byref(work))
    return (A, int(work.value)) if return_work else A


def attention_backward(offsets, H, dh, q, k, v, dA, spec: AttnSpec, return_work=False, return_abs=False):
    """(dQ, dK, dV, dpos, dts) — exact gradient of attention_forward.  With return_abs also
    (dpos_abs, dts_abs): the sums of |ds| per table entry, the scale of the summation error
    bound of these cancelling sums (reading R15b)."""
    lib = _load()
    offsets = np.ascontiguousarray(offsets, dtype=np.int32)
    B = len(offsets) - 1
    q, k, v, dA = _f64(q), _f64(k), _f64(v), _f64(dA)
    T = int(offsets[-1])
    ld = q.shape[1]
    dQ = np.zeros((T, H * dh)); dK = np.zeros((T, H * dh)); dV = np.zeros((T, H * dh))
    pos = _f64(spec.pos_w)
    ts = _f64(spec.ts_w)
    dpos = None if pos is None else np.zeros(len(pos))
    dts = None if ts is None else np.zeros(len(ts))
    dpos_abs = None if (pos is None or not return_abs) else np.zeros(len(pos))
    dts_abs = None if (ts is None or not return_abs) else np.zeros(len(ts))
    t = None
    if ts is not None:
        t = np.ascontiguousarray(spec.timestamps, dtype=np.int64)
    work = ctypes.c_int64(0)
    lib.orc_attn_bwd(B, _ptr(offsets, ctypes.c_int32), H, dh,
                     _ptr(q, ctypes.c_double), _ptr(k, ctypes.c_double), _ptr(v, ctypes.c_double), ld,
                     _ptr(dA, ctypes.c_double), dA.shape[1],
                     spec.K1, spec.K2, float(spec.alpha), float(spec.N),
                     _ptr(pos, ctypes.c_double), 0 if pos is None else len(pos),
                     _ptr(ts, ctypes.c_double), 0 if ts is None else len(ts),
                     _ptr(t, ctypes.c_int64),
                     _ptr(dQ, ctypes.c_double), _ptr(dK, ctypes.c_double), _ptr(dV, ctypes.c_double), H * dh,
                     _ptr(dpos, ctypes.c_double), _ptr(dts, ctypes.c_double),
                     _ptr(dpos_abs, ctypes.c_double), _ptr(dts_abs, ctypes.c_double), ctypes.byref(work))
    out = (dQ, dK, dV, dpos, dts) + ((dpos_abs, dts_abs) if return_abs else ())
    return (out, int(work.value)) if return_work else out


# ----------------------------------------------------------------------------
# elementwise pieces (§3: "phi1 and phi2 are SiLU"; Eq. 1 / Eq. 4 Norm = LayerNorm, R9)
# ----------------------------------------------------------------------------
def silu(x):
    return x / (1.0 + np.exp(-x))


def silu_grad(x):
    s = 1.0 / (1.0 + np.exp(-x))
    return s * (1.0 + x * (1.0 - s))


def layer_norm(x, w, b, eps):
    """LayerNorm over the last dim, biased variance (R9).  Returns (y, mu, rstd)."""
    mu = x.mean(axis=1, keepdims=True)
    var = ((x - mu) ** 2).mean(axis=1, keepdims=True)
    rstd = 1.0 / np.sqrt(var + eps)
    y = (x - mu) * rstd * w[None, :] + b[None, :]
    return y, mu[:, 0], rstd[:, 0]


def layer_norm_backward(g, x, mu, rstd, w):
    """d/dx, d/dw, d/db of layer_norm for upstream gradient g."""
    xt = (x - mu[:, None]) * rstd[:, None]
    gh = g * w[None, :]
    dx = rstd[:, None] * (gh - gh.mean(axis=1, keepdims=True)
                          - xt * (gh * xt).mean(axis=1, keepdims=True))
    return dx, (g * xt).sum(axis=0), g.sum(axis=0)


# ----------------------------------------------------------------------------
# the layer (Eqs. 1-5, Listing 1)
# ----------------------------------------------------------------------------
@dataclass
class LayerParams:
    ln1_w: np.ndarray
    ln1_b: np.ndarray
    w1: np.ndarray            # [d, 4d], columns U|V|Q|K (Listing 1 split order, R11)
    ln2_w: np.ndarray
    ln2_b: np.ndarray
    w2: np.ndarray            # [d, d]
    b1: Optional[np.ndarray] = None   # [4d]
    b2: Optional[np.ndarray] = None   # [d]
    eps: float = 1e-6


def layer_forward(x, offsets, prm: LayerParams, H: int, spec: AttnSpec):
    """Eqs. 1-5 in Listing 1's order.  Returns (out, cache)."""
    x = _f64(x)
    d = x.shape[1]
    xh, mu1, rs1 = layer_norm(x, _f64(prm.ln1_w), _f64(prm.ln1_b), prm.eps)      # Eq. 1
    h = xh @ _f64(prm.w1)                                                         # f1 (Eq. 2)
    if prm.b1 is not None:
        h = h + _f64(prm.b1)[None, :]
    s = silu(h)                                                                   # phi1
    U, V, Q, K = s[:, :d], s[:, d:2 * d], s[:, 2 * d:3 * d], s[:, 3 * d:]
    A = attention_forward(offsets, H, d // H, Q, K, V, spec)                      # Eq. 3
    Ah, mu2, rs2 = layer_norm(A, _f64(prm.ln2_w), _f64(prm.ln2_b), prm.eps)      # Norm(A)
    Y = Ah * U                                                                    # (.) U, Eq. 4
    out = Y @ _f64(prm.w2) + x                                                    # f2 + residual, Eqs. 4-5
    if prm.b2 is not None:
        out = out + _f64(prm.b2)[None, :]
    cache = dict(x=x, xh=xh, mu1=mu1, rs1=rs1, h=h, U=U, V=V, Q=Q, K=K, A=A,
                 Ah=Ah, mu2=mu2, rs2=rs2, Y=Y)
    return out, cache


def layer_backward(dout, offsets, prm: LayerParams, H: int, spec: AttnSpec, cache=None, x=None, rab_abs=False):
    """Exact gradient of layer_forward for the loss sum(dout * out).

    Returns (dx, grads) with grads keys ln1_w, ln1_b, w1, b1, ln2_w, ln2_b, w2, b2,
    pos_w, ts_w (with rab_abs also pos_w_abs, ts_w_abs: the sums of |ds| per entry, R15b).
    Parameter gradients are sums over all tokens."""
    if cache is None:
        _, cache = layer_forward(x, offsets, prm, H, spec)
    dout = _f64(dout)
    d = dout.shape[1]
    c = cache
    g = {}
    g["w2"] = c["Y"].T @ dout                                   # d_linear_w_2
    g["b2"] = dout.sum(axis=0)
    dY = dout @ _f64(prm.w2).T                                  # dy
    dAh = dY * c["U"]                                           # gated_norm_backward
    dU = dY * c["Ah"]
    dA, g["ln2_w"], g["ln2_b"] = layer_norm_backward(dAh, c["A"], c["mu2"], c["rs2"], _f64(prm.ln2_w))
    ab = attention_backward(                                    # attention_backward
        offsets, H, d // H, c["Q"], c["K"], c["V"], dA, spec, return_abs=rab_abs)
    dQ, dK, dV, g["pos_w"], g["ts_w"] = ab[:5]
    if rab_abs:
        g["pos_w_abs"], g["ts_w_abs"] = ab[5:]
    dS = np.concatenate([dU, dV, dQ, dK], axis=1)               # duqkv
    dH = dS * silu_grad(c["h"])                                 # silu_backward
    g["w1"] = c["xh"].T @ dH                                    # d_linear_w_1
    g["b1"] = dH.sum(axis=0)
    dxh = dH @ _f64(prm.w1).T                                   # d_normed_x
    dx, g["ln1_w"], g["ln1_b"] = layer_norm_backward(dxh, c["x"], c["mu1"], c["rs1"], _f64(prm.ln1_w))
    dx = dx + dout                                              # dx += dout
    return dx, g


# ----------------------------------------------------------------------------
# token-balanced partitioner (load notion of P:112)
# ----------------------------------------------------------------------------
def seq_cost(L: int, d: int, H: int, K1: int, K2: int) -> float:
    """c(L) = 4 (2 L d 4d) + 3 (2 L d d) + 14 d_h H nnz(L): the flops one layer step spends on a
    length-L sequence.  f1-shaped GEMMs: forward f1 (Eq. 2), the remat f1
    (P:187), dW1 and dx^ (Listing 1); f2-shaped: forward f2 (Eq. 4), dY and dW2
    (P:563-567); attention 4 d_h forward + 10 d_h backward flops per allowed pair-head."""
    dh = d // H
    return 4.0 * (2.0 * L * d * 4 * d) + 3.0 * (2.0 * L * d * d) + 14.0 * dh * H * mask_nnz(L, K1, K2)


def partition_lpt(lengths, world: int, d: int, H: int, K1: int, K2: int):
    """Longest-processing-time-first: sort by (cost desc, seq id asc); give each
    sequence to the least-loaded rank, lowest rank id on ties.  Step by step."""
    costs = [seq_cost(int(L), d, H, K1, K2) for L in lengths]
    order = sorted(range(len(lengths)), key=lambda i: (-costs[i], i))
    load = [0.0] * world
    owner = [-1] * len(lengths)
    for i in order:
        best = 0
        for r in range(1, world):
            if load[r] < load[best]:
                best = r
        owner[i] = best
        load[best] += costs[i]
    return owner, load


# ----------------------------------------------------------------------------
# NEXT-2: FP8 projections (§4.2.2 "Mixed-Precision Training and
# Inference", App. E.1).  "We execute both GEMMs in FP8, while
# preserving all remaining operations in BF16"; the row-wise scale and
# quantisation are computed with the preceding layer norms (Fig. fp8).
# Readings R17-R20: E4M3FN codes, round-to-nearest-even with
# saturation at 448; activation scale per row s_r = amax_r / 448 (1 for an
# all-zero row), weight scale per output column; the oracle quantises by the
# plain definition in fp64 (R19: the kernel's fp32 decision may pick the
# adjacent code where x / s is within fp32 noise of a midpoint).
# ----------------------------------------------------------------------------
E4M3_MAX = 448.0


def e4m3_round(v):
    """Nearest E4M3FN value (1 sign, 4 exponent bits with bias 7, 3 mantissa bits;
    normals 2^-6 .. 448, subnormals k 2^-9), ties to even, |result| <= 448 (R17)."""
    v = np.asarray(v, np.float64)
    a = np.abs(v)
    e = np.floor(np.log2(np.where(a > 0, a, 1.0)))
    e = np.maximum(e, -6.0)                 # below 2^-6 the spacing stays 2^-9 (subnormals)
    ulp = np.exp2(e - 3.0)                  # 3 mantissa bits
    r = np.round(a / ulp) * ulp             # np.round: half to even; a / ulp is exact
    r = np.minimum(r, E4M3_MAX)             # satfinite
    return np.where(a > 0, np.copysign(r, v), 0.0)


def quant_rows_e4m3(x):
    """Row-wise FP8 quantisation (R18): the plain definition in fp64,
    s_r = amax_r / 448 (1 for an all-zero row) and q = RNE_e4m3(x / s_r).  x [R, C] ->
    (q [R, C] float64 holding E4M3 values, s [R] float64), x ~= q * s[:, None].
    (The kernel takes the same steps in fp32; its codes may differ from these only where
    x / s sits within fp32 rounding of an E4M3 midpoint -- reading R19.)"""
    x = np.asarray(x, np.float64)
    amax = np.abs(x).max(axis=1) if x.shape[1] else np.zeros(x.shape[0])
    s = np.where(amax > 0, amax / E4M3_MAX, 1.0)
    return e4m3_round(x / s[:, None]), s


def quant_weight_e4m3(w):
    """Per-output-column quantisation of a weight W [K, N] (R18): returns (qT [N, K]
    E4M3 values, s [N]) with W[:, n] ~= qT[n, :] * s[n]."""
    return quant_rows_e4m3(np.asarray(w, np.float64).T)


def gemm_fp8(qa, sa, qbT, sb):
    """Row-wise scaled FP8 GEMM: D = diag(sa) (qa qbT^T) diag(sb), fp64
    accumulation of the exact code products."""
    return (np.asarray(qa, np.float64) @ np.asarray(qbT, np.float64).T) * np.asarray(sa)[:, None] \
        * np.asarray(sb)[None, :]


def layer_forward_fp8(x, offsets, prm: LayerParams, H: int, spec: AttnSpec):
    """Eqs. 1-5 with both projections in FP8: x^ = Norm(x) quantised per row
    (P:164); h = FP8GEMM(x^, W1) + b1; attention and the gated norm as in
    layer_forward; Y quantised per row; out = FP8GEMM(Y, W2) + b2 + x (the 2-D bias
    fused into the GEMM).  Returns (out, cache)."""
    x = _f64(x)
    d = x.shape[1]
    xh, mu1, rs1 = layer_norm(x, _f64(prm.ln1_w), _f64(prm.ln1_b), prm.eps)      # Eq. 1
    qx, sx = quant_rows_e4m3(xh)                                                  # fused quant
    qw1, sw1 = quant_weight_e4m3(prm.w1)
    h = gemm_fp8(qx, sx, qw1, sw1)                                                # f1 in FP8 (Eq. 2)
    if prm.b1 is not None:
        h = h + _f64(prm.b1)[None, :]
    s = silu(h)
    U, V, Q, K = s[:, :d], s[:, d:2 * d], s[:, 2 * d:3 * d], s[:, 3 * d:]
    A = attention_forward(offsets, H, d // H, Q, K, V, spec)                      # Eq. 3
    Ah, mu2, rs2 = layer_norm(A, _f64(prm.ln2_w), _f64(prm.ln2_b), prm.eps)
    Y = Ah * U                                                                    # Eq. 4 inner
    qy, sy = quant_rows_e4m3(Y)                                                   # fused quant
    qw2, sw2 = quant_weight_e4m3(prm.w2)
    out = gemm_fp8(qy, sy, qw2, sw2) + x                                          # f2 + 2-D bias
    if prm.b2 is not None:
        out = out + _f64(prm.b2)[None, :]
    cache = dict(xh=xh, qx=qx, sx=sx, h=h, U=U, V=V, Q=Q, K=K, A=A, Y=Y, qy=qy, sy=sy,
                 mu1=mu1, rs1=rs1, mu2=mu2, rs2=rs2)
    return out, cache
