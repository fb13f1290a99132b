"""Thin ctypes binding of libuhstu (include/uhstu.h).

Argument marshalling only: every step of the hot path runs in the library's CUDA
kernels.  PyTorch provides device memory and the current stream.  If the shared
library is missing this module raises on first use — there is no CPU fallback.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libuhstu.so")
WINDOW_FULL = 2**31 - 1

BF16, F32 = 0, 1
_DT = {torch.bfloat16: BF16, torch.float32: F32}

_lib = None


class UhError(RuntimeError):
    def __init__(self, status: int, name: str, detail: str):
        super().__init__(f"{name}: {detail}")
        self.status = status
        self.name = name


# ----------------------------------------------------------------------------- structs
class Jagged(ctypes.Structure):
    _fields_ = [("num_seqs", ctypes.c_int32), ("max_len", ctypes.c_int32), ("total_tokens", ctypes.c_int64),
                ("offsets", ctypes.c_void_p), ("host_offsets", ctypes.POINTER(ctypes.c_int32))]


class Mask(ctypes.Structure):
    _fields_ = [("window", ctypes.c_int32), ("n_global", ctypes.c_int32)]


class AttnDesc(ctypes.Structure):
    _fields_ = [("num_heads", ctypes.c_int32), ("head_dim", ctypes.c_int32), ("alpha", ctypes.c_float),
                ("norm_n", ctypes.c_float), ("pos_bias", ctypes.c_void_p), ("pos_bias_len", ctypes.c_int32),
                ("time_bias", ctypes.c_void_p), ("time_bias_len", ctypes.c_int32), ("timestamps", ctypes.c_void_p)]


class LayerParams(ctypes.Structure):
    _fields_ = [("ln1_w", ctypes.c_void_p), ("ln1_b", ctypes.c_void_p), ("w1", ctypes.c_void_p),
                ("b1", ctypes.c_void_p), ("ln2_w", ctypes.c_void_p), ("ln2_b", ctypes.c_void_p),
                ("w2", ctypes.c_void_p), ("b2", ctypes.c_void_p), ("attn", AttnDesc), ("eps", ctypes.c_float)]


class LayerSaved(ctypes.Structure):
    _fields_ = [("attn", ctypes.c_void_p), ("ln1_mean", ctypes.c_void_p), ("ln1_rstd", ctypes.c_void_p),
                ("ln2_mean", ctypes.c_void_p), ("ln2_rstd", ctypes.c_void_p), ("fingerprint", ctypes.c_uint64)]


class LayerGrads(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in
                ("ln1_w", "ln1_b", "w1", "b1", "ln2_w", "ln2_b", "w2", "b2", "pos_bias", "time_bias")]


class MotBranch(ctypes.Structure):
    """uh_mot_branch (include/uhstu_mot.h)."""
    _fields_ = [("jag", ctypes.POINTER(Jagged)), ("x", ctypes.c_void_p), ("ld", ctypes.c_int64)]


class Fp8Weights(ctypes.Structure):
    """uh_fp8_weights (include/uhstu_fp8.h)."""
    _fields_ = [("w1t", ctypes.c_void_p), ("s1", ctypes.c_void_p), ("w2t", ctypes.c_void_p), ("s2", ctypes.c_void_p)]


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"libuhstu not built ({LIB_PATH} missing): run __graft_entry__.build()")
        L = ctypes.CDLL(LIB_PATH)
        P = ctypes.POINTER
        vp, i32, i64, sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t
        L.uh_status_string.restype = ctypes.c_char_p
        L.uh_status_string.argtypes = [ctypes.c_int]
        L.uh_last_error.restype = ctypes.c_char_p
        L.uh_abi_version.restype = ctypes.c_int
        L.uh_mask_nnz.restype = i64
        L.uh_mask_nnz.argtypes = [Mask, i64]
        L.uh_batch_nnz.restype = i64
        L.uh_batch_nnz.argtypes = [P(Jagged), Mask]
        L.uh_attn_workspace_bytes.argtypes = [P(Jagged), Mask, P(AttnDesc), ctypes.c_int, ctypes.c_int, P(sz)]
        L.uh_attn_fwd.argtypes = [P(Jagged), Mask, P(AttnDesc), ctypes.c_int, vp, vp, vp, i64, vp, i64, vp, sz, vp]
        L.uh_attn_bwd.argtypes = [P(Jagged), Mask, P(AttnDesc), ctypes.c_int, vp, vp, vp, i64, vp, i64,
                                  vp, vp, vp, i64, vp, vp, vp, sz, vp]
        L.uh_layer_workspace_bytes.argtypes = [P(Jagged), Mask, P(LayerParams), ctypes.c_int, ctypes.c_int, P(sz)]
        L.uh_layer_fwd.argtypes = [P(Jagged), Mask, P(LayerParams), ctypes.c_int, vp, vp, P(LayerSaved), vp, sz, vp]
        L.uh_layer_bwd.argtypes = [P(Jagged), Mask, P(LayerParams), ctypes.c_int, vp, P(LayerSaved), vp, vp,
                                   P(LayerGrads), ctypes.c_int, vp, sz, vp]
        L.uh_jagged_gather.argtypes = [P(Jagged), P(i32), i32, vp, i64, i64, i32, vp, P(i32), vp, vp]
        L.uh_jagged_slice_latest.argtypes = [P(Jagged), i32, vp, i64, i64, i32, vp, P(i32), vp, vp]
        L.uh_jagged_to_padded.argtypes = [P(Jagged), vp, i64, i32, i32, vp, vp]
        L.uh_padded_to_jagged.argtypes = [P(Jagged), vp, i64, i32, i32, vp, vp]
        L.uh_partition_lpt.argtypes = [P(i32), i32, i32, Mask, i32, i32, P(i32), P(ctypes.c_double)]
        for f in ("uh_attn_workspace_bytes", "uh_attn_fwd", "uh_attn_bwd", "uh_layer_workspace_bytes",
                  "uh_layer_fwd", "uh_layer_bwd", "uh_jagged_gather", "uh_jagged_slice_latest",
                  "uh_jagged_to_padded", "uh_padded_to_jagged", "uh_partition_lpt"):
            getattr(L, f).restype = ctypes.c_int
        L.uh_test_gemm.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, vp, i64, ctypes.c_int, vp, i64,
                                   ctypes.c_int, ctypes.c_int, vp, i64, vp, i64, vp, vp, i64, ctypes.c_int,
                                   ctypes.c_int, vp]
        L.uh_test_gemm.restype = ctypes.c_int
        L.uh_test_launch_count.restype = ctypes.c_longlong
        # NEXT-2: FP8 projections (include/uhstu_fp8.h)
        u8p = ctypes.c_void_p
        L.uh_ln_fwd_fp8.argtypes = [i64, ctypes.c_int, vp, i64, vp, vp, ctypes.c_float, u8p, i64, vp, vp, vp, vp]
        L.uh_gated_norm_fwd_fp8.argtypes = [i64, ctypes.c_int, vp, i64, vp, i64, vp, vp, ctypes.c_float, u8p, i64,
                                            vp, vp, vp, vp]
        L.uh_quant_weight_fp8.argtypes = [ctypes.c_int, ctypes.c_int, vp, i64, u8p, i64, vp, vp]
        L.uh_gemm_fp8.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, u8p, i64, vp, u8p, i64, vp, ctypes.c_int,
                                  vp, i64, vp, vp, i64, vp]
        L.uh_layer_fwd_fp8.argtypes = [P(Jagged), Mask, P(LayerParams), P(Fp8Weights), vp, vp, P(LayerSaved), vp,
                                       sz, vp]
        for f in ("uh_ln_fwd_fp8", "uh_gated_norm_fwd_fp8", "uh_quant_weight_fp8", "uh_gemm_fp8",
                  "uh_layer_fwd_fp8"):
            getattr(L, f).restype = ctypes.c_int
        # NEXT-3: LBSL (include/uhstu_lbsl.h)
        u64, f64, P32 = ctypes.c_uint64, ctypes.c_double, P(i32)
        L.uh_lbsl_select.argtypes = [P32, i32, i32, f64, f64, i32, u64, i32, i64, P32, P32, P(f64)]
        L.uh_lbsl_subset.argtypes = [i32, i32, u64, i32, i64, i32, P32]
        L.uh_lbsl_rows.argtypes = [P32, i32, P32, P32, u64, i32, i64, P32, P32]
        L.uh_gather_rows.argtypes = [vp, i64, vp, i64, i64, i32, vp, i64, vp]
        for f in ("uh_lbsl_select", "uh_lbsl_subset", "uh_lbsl_rows", "uh_gather_rows"):
            getattr(L, f).restype = ctypes.c_int
        # NEXT-4: MoT fusion (include/uhstu_mot.h)
        L.uh_mot_workspace_bytes.argtypes = [i32, P(MotBranch), i32, i32, ctypes.c_int, ctypes.c_int, P(sz)]
        L.uh_mot_fuse_fwd.argtypes = [i32, P(MotBranch), i32, i32, ctypes.c_int, vp, vp, vp, vp, sz, vp]
        L.uh_mot_fuse_bwd.argtypes = [i32, P(MotBranch), i32, i32, ctypes.c_int, vp, vp, vp, vp, ctypes.c_int,
                                      P(vp), P(i64), vp, sz, vp]
        for f in ("uh_mot_workspace_bytes", "uh_mot_fuse_fwd", "uh_mot_fuse_bwd"):
            getattr(L, f).restype = ctypes.c_int
        if L.uh_abi_version() != 1:
            raise RuntimeError("libuhstu ABI version mismatch")
        _lib = L
    return _lib


def launch_count() -> int:
    """Kernels launched by libuhstu so far in this process."""
    return int(lib().uh_test_launch_count())


def exported_symbols() -> list:
    return ["uh_status_string", "uh_last_error", "uh_abi_version", "uh_mask_nnz", "uh_batch_nnz",
            "uh_attn_workspace_bytes", "uh_attn_fwd", "uh_attn_bwd", "uh_layer_workspace_bytes", "uh_layer_fwd",
            "uh_layer_bwd", "uh_jagged_gather", "uh_jagged_slice_latest", "uh_jagged_to_padded",
            "uh_padded_to_jagged", "uh_partition_lpt", "uh_ln_fwd_fp8", "uh_gated_norm_fwd_fp8",
            "uh_quant_weight_fp8", "uh_gemm_fp8", "uh_layer_fwd_fp8", "uh_lbsl_select", "uh_lbsl_subset",
            "uh_lbsl_rows", "uh_gather_rows", "uh_mot_workspace_bytes", "uh_mot_fuse_fwd", "uh_mot_fuse_bwd"]


def _check(st: int):
    if st != 0:
        L = lib()
        raise UhError(st, L.uh_status_string(st).decode(), L.uh_last_error().decode())


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


# ----------------------------------------------------------------------------- jagged batch
class JaggedBatch:
    """Host + device copies of the offsets of a jagged batch."""

    def __init__(self, offsets, device="cuda"):
        off = np.ascontiguousarray(np.asarray(offsets, dtype=np.int32))
        self.host = off
        self.lengths = np.diff(off)
        self.B = len(off) - 1
        self.T = int(off[-1]) if len(off) else 0
        self.max_len = int(self.lengths.max()) if self.B > 0 else 0
        self.dev = torch.from_numpy(off.copy()).to(device) if device is not None else None
        self.c = Jagged(self.B, self.max_len, self.T,
                        ctypes.c_void_p(self.dev.data_ptr()) if self.dev is not None else None,
                        self.host.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)))

    @staticmethod
    def from_lengths(lengths, device="cuda"):
        off = np.zeros(len(lengths) + 1, np.int32)
        off[1:] = np.cumsum(lengths)
        return JaggedBatch(off, device)


def mask(window: int = WINDOW_FULL, n_global: int = 0) -> Mask:
    return Mask(int(min(window, WINDOW_FULL)), int(n_global))


@dataclass
class Attn:
    """Attention descriptor (uh_attn_desc) with the tensors it points to kept alive."""
    num_heads: int
    head_dim: int
    alpha: float = 1.0
    norm_n: float = 1.0
    pos_bias: Optional[torch.Tensor] = None      # fp32 [P]
    time_bias: Optional[torch.Tensor] = None     # fp32 [NB]
    timestamps: Optional[torch.Tensor] = None    # int64 [T]

    def c(self) -> AttnDesc:
        return AttnDesc(self.num_heads, self.head_dim, self.alpha, self.norm_n,
                        _ptr(self.pos_bias), 0 if self.pos_bias is None else self.pos_bias.numel(),
                        _ptr(self.time_bias), 0 if self.time_bias is None else self.time_bias.numel(),
                        _ptr(self.timestamps))


def mask_nnz(m: Mask, L: int) -> int:
    return int(lib().uh_mask_nnz(m, L))


def batch_nnz(jag: JaggedBatch, m: Mask) -> int:
    return int(lib().uh_batch_nnz(ctypes.byref(jag.c), m))


def _dtype_code(t: torch.Tensor) -> int:
    if t.dtype not in _DT:
        raise TypeError(f"unsupported dtype {t.dtype}")
    return _DT[t.dtype]


# ----------------------------------------------------------------------------- attention
def attn_workspace_bytes(jag, m, desc: Attn, dtype: int, backward: bool) -> int:
    n = ctypes.c_size_t(0)
    d = desc.c()
    _check(lib().uh_attn_workspace_bytes(ctypes.byref(jag.c), m, ctypes.byref(d), dtype, int(backward), ctypes.byref(n)))
    return int(n.value)


def _ws(nbytes: int, device) -> torch.Tensor:
    return torch.empty(max(nbytes, 256), dtype=torch.uint8, device=device)


def _rows(name: str, *ts) -> int:
    """The C ABI takes ONE row stride for a group of [T, width] operands (q/k/v, or dq/dk/dv):
    each must be a 2-D row-major view (unit column stride) and all must share the row stride."""
    ld = None
    for t in ts:
        if t.dim() != 2 or t.stride(1) != 1:
            raise ValueError(f"{name}: expected 2-D row-major views with unit column stride")
        if ld is not None and t.stride(0) != ld:
            raise ValueError(f"{name}: all operands must share one row stride (got {ld} and {t.stride(0)})")
        ld = t.stride(0)
    return ld


def attn_fwd(jag: JaggedBatch, m: Mask, desc: Attn, q, k, v, out=None, ws=None):
    """A = attention(Q, K, V) for the jagged batch; q/k/v may be column views of one buffer."""
    dt = _dtype_code(q)
    ld_qkv = _rows("q/k/v", q, k, v)
    width = desc.num_heads * desc.head_dim
    if out is None:
        out = torch.empty(q.shape[0], width, dtype=q.dtype, device=q.device)
    d = desc.c()
    if ws is None:
        ws = _ws(attn_workspace_bytes(jag, m, desc, dt, False), q.device)
    _rows("out", out)
    _check(lib().uh_attn_fwd(ctypes.byref(jag.c), m, ctypes.byref(d), dt, _ptr(q), _ptr(k), _ptr(v), ld_qkv,
                             _ptr(out), out.stride(0), _ptr(ws), ws.numel(), _stream()))
    return out


def attn_bwd(jag: JaggedBatch, m: Mask, desc: Attn, q, k, v, dout, dq=None, dk=None, dv=None,
             dpos=None, dts=None, ws=None):
    """(dQ, dK, dV, dpos, dts); dpos/dts are fp32 and accumulated into if given."""
    dt = _dtype_code(q)
    width = desc.num_heads * desc.head_dim
    mk = lambda: torch.empty(q.shape[0], width, dtype=q.dtype, device=q.device)
    if dq is None and dk is None and dv is None:
        g = torch.empty(q.shape[0], 3 * width, dtype=q.dtype, device=q.device)
        dq, dk, dv = g[:, :width], g[:, width:2 * width], g[:, 2 * width:]
    dq = mk() if dq is None else dq
    dk = mk() if dk is None else dk
    dv = mk() if dv is None else dv
    if dpos is None and desc.pos_bias is not None:
        dpos = torch.zeros_like(desc.pos_bias)
    if dts is None and desc.time_bias is not None:
        dts = torch.zeros_like(desc.time_bias)
    ld_qkv = _rows("q/k/v", q, k, v)
    ld_grad = _rows("dq/dk/dv", dq, dk, dv)
    _rows("dout", dout)
    d = desc.c()
    if ws is None:
        ws = _ws(attn_workspace_bytes(jag, m, desc, dt, True), q.device)
    _check(lib().uh_attn_bwd(ctypes.byref(jag.c), m, ctypes.byref(d), dt, _ptr(q), _ptr(k), _ptr(v), ld_qkv,
                             _ptr(dout), dout.stride(0), _ptr(dq), _ptr(dk), _ptr(dv), ld_grad,
                             _ptr(dpos), _ptr(dts), _ptr(ws), ws.numel(), _stream()))
    return dq, dk, dv, dpos, dts


# ----------------------------------------------------------------------------- layer
@dataclass
class Params:
    """One HSTU layer's parameters (Listing 1 signature): LN1, W1 [d,4d] (+b1), LN2, W2 [d,d] (+b2)."""
    ln1_w: torch.Tensor
    ln1_b: torch.Tensor
    w1: torch.Tensor
    ln2_w: torch.Tensor
    ln2_b: torch.Tensor
    w2: torch.Tensor
    b1: Optional[torch.Tensor] = None
    b2: Optional[torch.Tensor] = None
    eps: float = 1e-6

    def c(self, attn: Attn) -> LayerParams:
        return LayerParams(_ptr(self.ln1_w), _ptr(self.ln1_b), _ptr(self.w1), _ptr(self.b1), _ptr(self.ln2_w),
                           _ptr(self.ln2_b), _ptr(self.w2), _ptr(self.b2), attn.c(), self.eps)


@dataclass
class Saved:
    attn: torch.Tensor
    ln1_mean: torch.Tensor
    ln1_rstd: torch.Tensor
    ln2_mean: torch.Tensor
    ln2_rstd: torch.Tensor
    fingerprint: int = 0   # written by the forward, checked by the backward (uh_layer_saved)

    def c(self) -> LayerSaved:
        return LayerSaved(_ptr(self.attn), _ptr(self.ln1_mean), _ptr(self.ln1_rstd), _ptr(self.ln2_mean),
                          _ptr(self.ln2_rstd), self.fingerprint)

    def nbytes(self) -> int:
        return sum(t.numel() * t.element_size() for t in (self.attn, self.ln1_mean, self.ln1_rstd,
                                                          self.ln2_mean, self.ln2_rstd))


def layer_workspace_bytes(jag, m, prm: Params, attn: Attn, dtype: int, backward: bool) -> int:
    n = ctypes.c_size_t(0)
    p = prm.c(attn)
    _check(lib().uh_layer_workspace_bytes(ctypes.byref(jag.c), m, ctypes.byref(p), dtype, int(backward),
                                          ctypes.byref(n)))
    return int(n.value)


def alloc_saved(x: torch.Tensor) -> Saved:
    f = lambda: torch.empty(x.shape[0], dtype=torch.float32, device=x.device)
    return Saved(torch.empty_like(x), f(), f(), f(), f())


def layer_fwd(jag, m, prm: Params, attn: Attn, x, save: bool = True, out=None, ws=None, saved: Optional[Saved] = None):
    """out = HSTU layer(x) (Eqs. 1-5); returns (out, saved) — saved is the remat set for layer_bwd."""
    dt = _dtype_code(x)
    out = torch.empty_like(x) if out is None else out
    if save and saved is None:
        saved = alloc_saved(x)
    if not save:
        saved = None
    p = prm.c(attn)
    if ws is None:
        ws = _ws(layer_workspace_bytes(jag, m, prm, attn, dt, False), x.device)
    sc = saved.c() if saved is not None else None
    _check(lib().uh_layer_fwd(ctypes.byref(jag.c), m, ctypes.byref(p), dt, _ptr(x), _ptr(out),
                              ctypes.byref(sc) if sc is not None else None, _ptr(ws), ws.numel(), _stream()))
    if saved is not None:
        saved.fingerprint = int(sc.fingerprint)
    return out, saved


def layer_bwd(jag, m, prm: Params, attn: Attn, x, saved: Saved, dout, grads: Optional[dict] = None,
              accumulate: bool = False, dx=None, ws=None):
    """Returns (dx, grads) — grads: fp32 tensors keyed like Params (+ pos_bias, time_bias)."""
    dt = _dtype_code(x)
    dx = torch.empty_like(x) if dx is None else dx
    if grads is None:
        z = lambda t: None if t is None else torch.zeros(t.shape, dtype=torch.float32, device=x.device)
        grads = dict(ln1_w=z(prm.ln1_w), ln1_b=z(prm.ln1_b), w1=z(prm.w1), b1=z(prm.b1), ln2_w=z(prm.ln2_w),
                     ln2_b=z(prm.ln2_b), w2=z(prm.w2), b2=z(prm.b2), pos_bias=z(attn.pos_bias),
                     time_bias=z(attn.time_bias))
    g = LayerGrads(*[_ptr(grads.get(n)) for n, _ in LayerGrads._fields_])
    p = prm.c(attn)
    sc = saved.c()
    if ws is None:
        ws = _ws(layer_workspace_bytes(jag, m, prm, attn, dt, True), x.device)
    _check(lib().uh_layer_bwd(ctypes.byref(jag.c), m, ctypes.byref(p), dt, _ptr(x), ctypes.byref(sc), _ptr(dout),
                              _ptr(dx), ctypes.byref(g), int(accumulate), _ptr(ws), ws.numel(), _stream()))
    return dx, grads


# ----------------------------------------------------------------------------- jagged ops
def _offsets_out(n: int):
    return np.zeros(n + 1, np.int32)


def jagged_gather(jag: JaggedBatch, seq_ids: Sequence[int], x: torch.Tensor):
    ids = np.ascontiguousarray(np.asarray(seq_ids, np.int32))
    n = len(ids)
    tot = int(sum(jag.lengths[i] for i in ids))
    y = torch.empty(tot, x.shape[1], dtype=x.dtype, device=x.device)
    off = _offsets_out(n)
    _check(lib().uh_jagged_gather(ctypes.byref(jag.c), ids.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), n,
                                  _ptr(x), x.stride(0), x.shape[1], x.element_size(), _ptr(y),
                                  off.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), None, _stream()))
    return y, JaggedBatch(off, x.device)


def jagged_slice_latest(jag: JaggedBatch, l_keep: int, x: torch.Tensor, out: Optional[torch.Tensor] = None):
    tot = int(np.minimum(jag.lengths, l_keep).sum())
    y = torch.empty(tot, x.shape[1], dtype=x.dtype, device=x.device) if out is None else out
    if y.shape[0] != tot or y.stride(1) != 1:
        raise ValueError("jagged_slice_latest: out must hold the kept rows, row-major")
    off = _offsets_out(jag.B)
    _check(lib().uh_jagged_slice_latest(ctypes.byref(jag.c), int(l_keep), _ptr(x), x.stride(0), x.shape[1],
                                        x.element_size(), _ptr(y), off.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                                        None, _stream()))
    return y, JaggedBatch(off, x.device)


def jagged_to_padded(jag: JaggedBatch, x: torch.Tensor, max_len: int):
    y = torch.empty(jag.B, max_len, x.shape[1], dtype=x.dtype, device=x.device)
    _check(lib().uh_jagged_to_padded(ctypes.byref(jag.c), _ptr(x), x.shape[1], x.element_size(), max_len, _ptr(y),
                                     _stream()))
    return y


def padded_to_jagged(jag: JaggedBatch, y: torch.Tensor):
    x = torch.empty(jag.T, y.shape[2], dtype=y.dtype, device=y.device)
    _check(lib().uh_padded_to_jagged(ctypes.byref(jag.c), _ptr(y), y.shape[2], y.element_size(), y.shape[1], _ptr(x),
                                     _stream()))
    return x


def test_gemm(A, B, a_mn: bool, b_mn: bool, epi: int, M: int, N: int, K: int, bias=None, resid=None,
              out0=None, out1=None, cta_pair: int = 0):
    """Test hook (include/uhstu_testing.h): the internal projection GEMM."""
    dt = _dtype_code(A)
    if out0 is None:
        out0 = torch.zeros(M, N, dtype=torch.float32 if epi == 2 else A.dtype, device=A.device)
    _check(lib().uh_test_gemm(M, N, K, _ptr(A), A.stride(0), int(a_mn), _ptr(B), B.stride(0), int(b_mn), epi,
                              _ptr(out0), out0.stride(0), _ptr(out1), 0 if out1 is None else out1.stride(0),
                              _ptr(bias), _ptr(resid), 0 if resid is None else resid.stride(0), dt, int(cta_pair),
                              _stream()))
    return out0, out1


# ----------------------------------------------------------------------------- partitioner
def partition_lpt(lengths, world: int, m: Mask, d: int, num_heads: int):
    L = np.ascontiguousarray(np.asarray(lengths, np.int32))
    owner = np.zeros(len(L), np.int32)
    cost = np.zeros(world, np.float64)
    _check(lib().uh_partition_lpt(L.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), len(L), world, m, d, num_heads,
                                  owner.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                                  cost.ctypes.data_as(ctypes.POINTER(ctypes.c_double))))
    return owner, cost


# ----------------------------------------------------------------------------- NEXT-2: FP8 projections
# (include/uhstu_fp8.h).  Codes are torch.uint8 tensors (E4M3 bit patterns).
def _u8(T, d, dev):
    return torch.empty(T, d, dtype=torch.uint8, device=dev)


def ln_fwd_fp8(x, w, b, eps=1e-6, q=None, scale=None, mean=None, rstd=None):
    """codes(LN(x)), row scales (and LN statistics when mean / rstd are given)."""
    T, d = x.shape
    q = _u8(T, d, x.device) if q is None else q
    scale = torch.empty(T, dtype=torch.float32, device=x.device) if scale is None else scale
    _check(lib().uh_ln_fwd_fp8(T, d, _ptr(x), x.stride(0), _ptr(w), _ptr(b), eps, _ptr(q), q.stride(0),
                               _ptr(scale), _ptr(mean), _ptr(rstd), _stream()))
    return q, scale


def gated_norm_fwd_fp8(A, U_, w, b, eps=1e-6, q=None, scale=None, mean=None, rstd=None):
    """codes(LN(A) (.) U), row scales."""
    T, d = A.shape
    q = _u8(T, d, A.device) if q is None else q
    scale = torch.empty(T, dtype=torch.float32, device=A.device) if scale is None else scale
    _check(lib().uh_gated_norm_fwd_fp8(T, d, _ptr(A), A.stride(0), _ptr(U_), U_.stride(0), _ptr(w), _ptr(b), eps,
                                       _ptr(q), q.stride(0), _ptr(scale), _ptr(mean), _ptr(rstd), _stream()))
    return q, scale


def quant_weight_fp8(W):
    """W bf16 [K, N] -> (W^T codes [N, K], per-column scales [N])."""
    K, N = W.shape
    qt = _u8(N, K, W.device)
    s = torch.empty(N, dtype=torch.float32, device=W.device)
    _check(lib().uh_quant_weight_fp8(K, N, _ptr(W), W.stride(0), _ptr(qt), qt.stride(0), _ptr(s), _stream()))
    return qt, s


def gemm_fp8(qa, sa, qb, sb, epi: int = 0, bias=None, resid=None, out=None):
    """out = diag(sa) (qa qb^T) diag(sb) (+ bias)(+ resid) (epi 0) or silu(...) (epi 1), bf16."""
    M, K = qa.shape
    N = qb.shape[0]
    out = torch.empty(M, N, dtype=torch.bfloat16, device=qa.device) if out is None else out
    _check(lib().uh_gemm_fp8(M, N, K, _ptr(qa), qa.stride(0), _ptr(sa), _ptr(qb), qb.stride(0), _ptr(sb), epi,
                             _ptr(out), out.stride(0), _ptr(bias), _ptr(resid),
                             0 if resid is None else resid.stride(0), _stream()))
    return out


def quant_layer_weights(prm: Params):
    """The layer's uh_fp8_weights (run once per weight update); returns (struct, keep-alive tensors)."""
    w1t, s1 = quant_weight_fp8(prm.w1)
    w2t, s2 = quant_weight_fp8(prm.w2)
    return Fp8Weights(_ptr(w1t), _ptr(s1), _ptr(w2t), _ptr(s2)), (w1t, s1, w2t, s2)


def layer_fwd_fp8(jag, m, prm: Params, attn: Attn, x, qw, save: bool = False, out=None, ws=None,
                  saved: Optional[Saved] = None):
    """out = HSTU layer(x) with both projections in FP8; qw from quant_layer_weights."""
    out = torch.empty_like(x) if out is None else out
    if save and saved is None:
        saved = alloc_saved(x)
    if not save:
        saved = None
    p = prm.c(attn)
    if ws is None:
        ws = _ws(layer_workspace_bytes(jag, m, prm, attn, BF16, False), x.device)
    sc = saved.c() if saved is not None else None
    st, _keep = qw
    _check(lib().uh_layer_fwd_fp8(ctypes.byref(jag.c), m, ctypes.byref(p), ctypes.byref(st), _ptr(x), _ptr(out),
                                  ctypes.byref(sc) if sc is not None else None, _ptr(ws), ws.numel(), _stream()))
    if saved is not None:
        saved.fingerprint = int(sc.fingerprint)
    return out, saved


# ----------------------------------------------------------------------------- NEXT-3: LBSL
# (include/uhstu_lbsl.h; Alg. 1).  Host arrays are numpy; the gather is on device.
def _i32p(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))


def lbsl_select(lengths, ell_sl: int, gamma: float, ell_bar: float, steady: bool, seed: int, rank: int, step: int):
    """Alg. 1 lines 4-20 for one rank: (decision[b], new_len[b], proxy load)."""
    n = np.ascontiguousarray(np.asarray(lengths, np.int32))
    dec = np.zeros(len(n), np.int32)
    new = np.zeros(len(n), np.int32)
    proxy = ctypes.c_double(0.0)
    _check(lib().uh_lbsl_select(_i32p(n), len(n), int(ell_sl), float(gamma), float(ell_bar), int(bool(steady)),
                                int(seed) & (2 ** 64 - 1), int(rank), int(step), _i32p(dec), _i32p(new),
                                ctypes.byref(proxy)))
    return dec, new, proxy.value


def lbsl_subset(n: int, tau: int, seed: int, rank: int, step: int, u: int):
    idx = np.zeros(max(tau, 0), np.int32)
    _check(lib().uh_lbsl_subset(int(n), int(tau), int(seed) & (2 ** 64 - 1), int(rank), int(step), int(u),
                                _i32p(idx)))
    return idx


def lbsl_rows(offsets, decision, new_len, seed: int, rank: int, step: int):
    """Source row of every kept token and the new offsets (host int32)."""
    off = np.ascontiguousarray(np.asarray(offsets, np.int32))
    dec = np.ascontiguousarray(np.asarray(decision, np.int32))
    nl = np.ascontiguousarray(np.asarray(new_len, np.int32))
    rows = np.zeros(int(nl.sum()), np.int32)
    new_off = np.zeros(len(off), np.int32)
    _check(lib().uh_lbsl_rows(_i32p(off), len(off) - 1, _i32p(dec), _i32p(nl), int(seed) & (2 ** 64 - 1), int(rank),
                              int(step), _i32p(rows), _i32p(new_off)))
    return rows, new_off


def gather_rows(rows_dev: torch.Tensor, x: torch.Tensor, out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """y[i] = x[rows[i]] on the device (uh_gather_rows)."""
    assert rows_dev.dtype == torch.int32 and rows_dev.is_cuda and x.is_cuda and x.dim() == 2
    n = rows_dev.numel()
    y = out if out is not None else torch.empty(n, x.shape[1], dtype=x.dtype, device=x.device)
    _check(lib().uh_gather_rows(_ptr(rows_dev), n, _ptr(x), x.stride(0), x.shape[1], x.element_size(), _ptr(y),
                                y.stride(0), _stream()))
    return y


# ----------------------------------------------------------------------------- NEXT-4: MoT fusion
def _mot_branches(jags: Sequence[JaggedBatch], xs: Sequence[torch.Tensor]):
    if len(jags) != len(xs):
        raise ValueError("one jagged batch per branch state")
    arr = (MotBranch * len(xs))()
    for i, (j, x) in enumerate(zip(jags, xs)):
        arr[i] = MotBranch(ctypes.pointer(j.c), _ptr(x), x.stride(0))
    return arr


def mot_workspace_bytes(jags, xs, n_cand: int, backward: bool) -> int:
    n = ctypes.c_size_t(0)
    br = _mot_branches(jags, xs)
    _check(lib().uh_mot_workspace_bytes(len(xs), br, int(n_cand), xs[0].shape[1], _dtype_code(xs[0]),
                                        int(backward), ctypes.byref(n)))
    return n.value


def mot_fuse_fwd(jags, xs, n_cand: int, w_f: torch.Tensor, b_f: Optional[torch.Tensor], out=None, ws=None):
    """E [B n_cand, d] = concat_k X_k[candidates] W_f + b_f (uh_mot_fuse_fwd)."""
    d = xs[0].shape[1]
    C = jags[0].B * n_cand
    e = torch.empty(C, d, dtype=xs[0].dtype, device=xs[0].device) if out is None else out
    if ws is None:
        ws = _ws(mot_workspace_bytes(jags, xs, n_cand, False), xs[0].device)
    _check(lib().uh_mot_fuse_fwd(len(xs), _mot_branches(jags, xs), int(n_cand), d, _dtype_code(xs[0]), _ptr(w_f),
                                 _ptr(b_f), _ptr(e), _ptr(ws), ws.numel(), _stream()))
    return e


def mot_fuse_bwd(jags, xs, n_cand: int, w_f: torch.Tensor, de: torch.Tensor, dw_f: torch.Tensor,
                 db_f: Optional[torch.Tensor] = None, accumulate: bool = False, dxs=None, ws=None):
    """dW_f, db_f (fp32, overwritten or accumulated) and each branch's output gradient dX_k
    (zero outside the candidate rows) -- uh_mot_fuse_bwd."""
    d = xs[0].shape[1]
    dxs = [torch.empty_like(x) for x in xs] if dxs is None else dxs
    ptrs = (ctypes.c_void_p * len(xs))(*[_ptr(t) for t in dxs])
    lds = (ctypes.c_int64 * len(xs))(*[t.stride(0) for t in dxs])
    if ws is None:
        ws = _ws(mot_workspace_bytes(jags, xs, n_cand, True), xs[0].device)
    _check(lib().uh_mot_fuse_bwd(len(xs), _mot_branches(jags, xs), int(n_cand), d, _dtype_code(xs[0]), _ptr(w_f),
                                 _ptr(de), _ptr(dw_f), _ptr(db_f), int(accumulate), ptrs, lds, _ptr(ws), ws.numel(),
                                 _stream()))
    return dxs
