"""Host-side tests of the C-ABI library (no GPU needed): the library loads, exports
every symbol include/*.h declares, validates arguments before launching anything,
and its host logic (closed-form nnz, LPT partitioner) matches the oracle."""
import ctypes
import os
import re
import subprocess
import sys

import numpy as np
import pytest

import oracle as O
from paper_2602_16986_b200 import uhstu as U

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    names = []
    for h in ("uhstu.h", "uhstu_testing.h", "uhstu_fp8.h", "uhstu_lbsl.h", "uhstu_mot.h"):
        txt = open(os.path.join(ROOT, "include", h)).read()
        names += re.findall(r"UH_API\s+[\w\s\*]+?\b(uh_\w+)\s*\(", txt)
    return sorted(set(names))


def test_library_exports_every_declared_symbol():
    syms = declared_symbols()
    assert len(syms) >= 22
    out = subprocess.run(["nm", "-D", "--defined-only", U.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\sT\s(uh_\w+)", out))
    missing = [s for s in syms if s not in exported]
    assert not missing, missing
    L = U.lib()
    for s in syms:
        assert hasattr(L, s)
    assert L.uh_abi_version() == 1


def test_mask_nnz_matches_oracle_enumeration():
    for L in (0, 1, 2, 17, 40, 64, 129, 300):
        for K1, K2 in ((16, 2), (0, 0), (1, 0), (5, 7), (U.WINDOW_FULL, 0), (128, 129), (300, 1)):
            okK1 = O.FULL if K1 == U.WINDOW_FULL else K1
            assert U.mask_nnz(U.mask(K1, K2), L) == O.mask_nnz(L, okK1, K2), (L, K1, K2)
    assert U.mask_nnz(U.mask(1024, 128), 16384) == 18226624


def test_partition_matches_oracle():
    rng = np.random.default_rng(0)
    for world in (1, 2, 3, 8):
        lengths = [int(x) for x in rng.integers(1, 700, size=23)] + [700, 700, 1]
        owner, cost = U.partition_lpt(lengths, world, U.mask(16, 2), 64, 2)
        o_owner, o_load = O.partition_lpt(lengths, world, 64, 2, 16, 2)
        assert list(owner) == o_owner
        assert np.allclose(cost, o_load, rtol=1e-12)


def test_partition_balances_cfg4_lengths():
    from paper_2602_16986_b200 import synth
    cfg = synth.config("cfg4", world=8)
    owner, cost = U.partition_lpt(cfg.lengths, 8, U.mask(cfg.K1, cfg.K2), cfg.d, cfg.H)
    assert sorted(set(owner.tolist())) == list(range(8))
    assert cost.max() / cost.mean() < 1.01


def _jag(offsets):
    return U.JaggedBatch(offsets, device=None)


def _status(fn):
    with pytest.raises(U.UhError) as e:
        fn()
    return e.value.name


def test_validation_errors_before_launch():
    desc = U.Attn(2, 32, norm_n=64.0)
    m = U.mask(16, 2)
    ok = _jag([0, 17, 57, 121])
    n = U.attn_workspace_bytes(ok, m, desc, U.F32, True)
    assert n > 0
    # bad offsets: decreasing -> DOMAIN; offsets[0] != 0 -> DIM
    bad = _jag([0, 17, 10, 121])
    assert _status(lambda: U.attn_workspace_bytes(bad, m, desc, U.F32, False)) == "UH_ERR_DOMAIN"
    bad0 = _jag([3, 17, 57, 121])
    assert _status(lambda: U.attn_workspace_bytes(bad0, m, desc, U.F32, False)) == "UH_ERR_DIM"
    wrong_max = _jag([0, 17, 57, 121]); wrong_max.c.max_len = 7
    assert _status(lambda: U.attn_workspace_bytes(wrong_max, m, desc, U.F32, False)) == "UH_ERR_DIM"
    assert _status(lambda: U.attn_workspace_bytes(ok, U.Mask(-1, 0), desc, U.F32, False)) == "UH_ERR_DOMAIN"
    assert _status(lambda: U.attn_workspace_bytes(ok, m, U.Attn(2, 48), U.F32, False)) == "UH_ERR_SHAPE"
    assert _status(lambda: U.attn_workspace_bytes(ok, m, U.Attn(2, 32), U.BF16, False)) == "UH_ERR_UNSUPPORTED"
    assert _status(lambda: U.attn_workspace_bytes(ok, m, U.Attn(2, 32, norm_n=0.0), U.F32, False)) == "UH_ERR_DOMAIN"
    # empty batch is a valid no-op
    assert U.attn_workspace_bytes(_jag([0]), m, desc, U.F32, False) >= 0


def test_null_and_alignment_checks_fwd():
    L = U.lib()
    jag = _jag([0, 17])
    jag.c.offsets = ctypes.c_void_p(0x1000)  # never dereferenced: checks fail first
    d = U.Attn(1, 32, norm_n=1.0).c()
    st = L.uh_attn_fwd(ctypes.byref(jag.c), U.mask(4, 0), ctypes.byref(d), U.F32, None, None, None, 32,
                       None, 32, None, 0, None)
    assert L.uh_status_string(st).decode() == "UH_ERR_NULL"
    st = L.uh_attn_fwd(ctypes.byref(jag.c), U.mask(4, 0), ctypes.byref(d), U.F32, ctypes.c_void_p(0x1008),
                       ctypes.c_void_p(0x1000), ctypes.c_void_p(0x1000), 32, ctypes.c_void_p(0x1000), 32, None, 0, None)
    assert L.uh_status_string(st).decode() == "UH_ERR_ALIGNMENT"
    st = L.uh_attn_fwd(ctypes.byref(jag.c), U.mask(4, 0), ctypes.byref(d), U.F32, ctypes.c_void_p(0x1000),
                       ctypes.c_void_p(0x1000), ctypes.c_void_p(0x1000), 30, ctypes.c_void_p(0x1000), 32, None, 0, None)
    assert L.uh_status_string(st).decode() == "UH_ERR_DIM"
    st = L.uh_attn_fwd(ctypes.byref(jag.c), U.mask(4, 0), ctypes.byref(d), U.F32, ctypes.c_void_p(0x1000),
                       ctypes.c_void_p(0x1000), ctypes.c_void_p(0x1000), 32, ctypes.c_void_p(0x1000), 32, None, 0, None)
    assert L.uh_status_string(st).decode() == "UH_ERR_WORKSPACE"


def test_layer_bwd_requires_saved_set():
    L = U.lib()
    jag = _jag([0, 17])
    jag.c.offsets = ctypes.c_void_p(0x1000)
    p = U.LayerParams()
    p.attn = U.Attn(2, 32, norm_n=1.0).c()
    for f in ("ln1_w", "ln1_b", "w1", "ln2_w", "ln2_b", "w2"):
        setattr(p, f, ctypes.c_void_p(0x1000))
    p.eps = 1e-6
    g = U.LayerGrads()
    st = L.uh_layer_bwd(ctypes.byref(jag.c), U.mask(4, 0), ctypes.byref(p), U.F32, ctypes.c_void_p(0x1000), None,
                        ctypes.c_void_p(0x1000), ctypes.c_void_p(0x1000), ctypes.byref(g), 0, None, 0, None)
    assert L.uh_status_string(st).decode() == "UH_ERR_CACHE_MISMATCH"


def test_bench_reference_arm_prints_one_json_line():
    """bench.py's contract: stdout carries exactly one JSON line (the oracle arm runs on CPU)."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--steps", "1", "--warmup", "3"], capture_output=True, text=True, cwd=ROOT, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, r.stdout[-2000:]
    import json
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["steps"] == 1 and d["warmup"] >= 3
    assert d["value"] > 0 and d["unit"] == "tokens/s" and d["n_gpus"] == 1
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0


def _layer_params_host(H=2, dh=32):
    p = U.LayerParams()
    p.attn = U.Attn(H, dh, norm_n=1.0).c()
    for f in ("ln1_w", "ln1_b", "w1", "ln2_w", "ln2_b", "w2"):
        setattr(p, f, ctypes.c_void_p(0x1000))
    p.eps = 1e-6
    return p


def test_layer_bwd_rejects_foreign_saved_set():
    """A saved set whose fingerprint was not written by a forward with the same batch, mask and
    descriptor is a CACHE_MISMATCH ("wrong cache variant"), checked before any launch."""
    L = U.lib()
    jag = _jag([0, 17])
    jag.c.offsets = ctypes.c_void_p(0x1000)
    p = _layer_params_host()
    g = U.LayerGrads(*[ctypes.c_void_p(0x1000)] * 10)
    fake = ctypes.c_void_p(0x1000)
    for fp in (0, 12345):
        s = U.LayerSaved(fake, fake, fake, fake, fake, fp)
        st = L.uh_layer_bwd(ctypes.byref(jag.c), U.mask(4, 0), ctypes.byref(p), U.F32, fake, ctypes.byref(s),
                            fake, fake, ctypes.byref(g), 0, None, 0, None)
        assert L.uh_status_string(st).decode() == "UH_ERR_CACHE_MISMATCH"


def test_layer_d_limit_checked_before_any_launch():
    """d above the row kernels' limit is UNSUPPORTED from the argument checks (nothing zeroed)."""
    L = U.lib()
    jag = _jag([0, 17])
    jag.c.offsets = ctypes.c_void_p(0x1000)
    p = _layer_params_host(H=9, dh=128)   # d = 1152 > 1024 (fp32 build)
    n = ctypes.c_size_t(0)
    st = L.uh_layer_workspace_bytes(ctypes.byref(jag.c), U.mask(4, 0), ctypes.byref(p), U.F32, 1, ctypes.byref(n))
    assert L.uh_status_string(st).decode() == "UH_ERR_UNSUPPORTED"


def test_binding_rejects_mismatched_qkv_strides():
    """The ABI takes one row stride for q/k/v; the binding refuses views that do not share it."""
    import torch
    q = torch.zeros(4, 64)
    k = torch.zeros(4, 128)[:, :64]
    with pytest.raises(ValueError):
        U._rows("q/k/v", q, k, q)
    with pytest.raises(ValueError):
        U._rows("dout", torch.zeros(64, 4).t())
    assert U._rows("q/k/v", q, q, q) == 64


def test_mot_validation_before_launch():
    """NEXT-4 (include/uhstu_mot.h): every argument check runs on the host before any launch."""
    L = U.lib()

    def branch_arr(jags, ld=64):
        arr = (U.MotBranch * len(jags))()
        for i, j in enumerate(jags):
            j.c.offsets = ctypes.c_void_p(0x1000)        # never dereferenced: checks fail first
            arr[i] = U.MotBranch(ctypes.pointer(j.c), ctypes.c_void_p(0x2000), ld)
        return arr

    def ws_status(jags, n_cand=2, d=64, dt=U.BF16, ld=64):
        n = ctypes.c_size_t(0)
        st = L.uh_mot_workspace_bytes(len(jags), branch_arr(jags, ld), n_cand, d, dt, 1, ctypes.byref(n))
        return L.uh_status_string(st).decode(), n.value

    a, b = _jag([0, 5, 9]), _jag([0, 3, 7])
    st, n = ws_status([a, b])
    assert st == "UH_OK" and n == 2 * ((2 * 2 * 2 * 64 * 2 + 255) // 256 * 256)
    assert ws_status([a, _jag([0, 3, 7, 9])])[0] == "UH_ERR_DIM"          # different user counts (R29)
    assert ws_status([a, _jag([0, 1, 7])])[0] == "UH_ERR_DIM"             # a sequence shorter than n_cand
    assert ws_status([a, b], n_cand=0)[0] == "UH_ERR_DOMAIN"
    assert ws_status([a] * 9)[0] == "UH_ERR_UNSUPPORTED"
    assert ws_status([a, b], d=96)[0] == "UH_ERR_SHAPE"                   # bf16 needs d % 64 == 0
    assert ws_status([a, b], ld=60)[0] == "UH_ERR_ALIGNMENT"
    arr = branch_arr([a, b])
    st = L.uh_mot_fuse_fwd(2, arr, 2, 64, U.BF16, None, None, ctypes.c_void_p(0x3000), None, 0, None)
    assert L.uh_status_string(st).decode() == "UH_ERR_NULL"
    st = L.uh_mot_fuse_fwd(2, arr, 2, 64, U.BF16, ctypes.c_void_p(0x3000), None, ctypes.c_void_p(0x3000), None, 0,
                           None)
    assert L.uh_status_string(st).decode() == "UH_ERR_WORKSPACE"
    dx = (ctypes.c_void_p * 2)(0x4000, 0x4008)
    lds = (ctypes.c_int64 * 2)(64, 64)
    st = L.uh_mot_fuse_bwd(2, arr, 2, 64, U.BF16, ctypes.c_void_p(0x3000), ctypes.c_void_p(0x3000),
                           ctypes.c_void_p(0x3000), None, 0, dx, lds, None, 0, None)
    assert L.uh_status_string(st).decode() == "UH_ERR_ALIGNMENT"
