"""Time the attention kernels alone at cfg3 for a few rab/mask variants (CUDA events)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2602_16986_b200 import synth  # noqa: E402
from paper_2602_16986_b200 import uhstu as U  # noqa: E402

if os.environ.get("UH_LIB"):   # experiment builds (tools/build_exp.py)
    U.LIB_PATH = os.path.join(ROOT, "paper_2602_16986_b200", "lib", os.environ["UH_LIB"])


def run(B=16, rab=True, K1=1024, K2=128, steps=10):
    cfg = synth.config("cfg3")
    lengths = [16384] * B
    jag = U.JaggedBatch.from_lengths(lengths)
    T, d = jag.T, cfg.d
    g = torch.Generator().manual_seed(0)
    buf = (torch.randn(T, 4 * d, generator=g) * (4.0 / 128) ** 0.25).to("cuda", torch.bfloat16)
    q, k, v = buf[:, 2 * d:3 * d], buf[:, 3 * d:], buf[:, d:2 * d]
    dA = torch.randn(T, d, generator=g).to("cuda", torch.bfloat16)
    pos, ts = synth.rab_tables(cfg)
    t = synth.timestamps(cfg.seed, lengths)
    use_pos, use_ts = rab in (True, "pos"), rab in (True, "ts")   # rab = True / False / "pos" / "ts"
    attn = U.Attn(4, 128, 1.0, float(cfg.N), torch.from_numpy(pos).cuda() if use_pos else None,
                  torch.from_numpy(ts).cuda() if use_ts else None, torch.from_numpy(t).cuda() if use_ts else None)
    m = U.mask(K1, K2)
    A = torch.empty(T, d, dtype=torch.bfloat16, device="cuda")
    gb = torch.empty(T, 3 * d, dtype=torch.bfloat16, device="cuda")
    wf = U._ws(U.attn_workspace_bytes(jag, m, attn, U.BF16, False), "cuda")
    wb = U._ws(U.attn_workspace_bytes(jag, m, attn, U.BF16, True), "cuda")
    fa = lambda: U.attn_fwd(jag, m, attn, q, k, v, out=A, ws=wf)
    fb = lambda: U.attn_bwd(jag, m, attn, q, k, v, dA, gb[:, :d], gb[:, d:2 * d], gb[:, 2 * d:], ws=wb)
    for _ in range(3):
        fa(); fb()
    res = {}
    for name, fn in (("fwd", fa), ("bwd", fb)):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        res[name] = e0.elapsed_time(e1) / steps
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(3):
            fa(); fb()
        torch.cuda.synchronize()
    ks = {}
    for e in prof.events():
        if e.device_type.name == "CUDA":
            ks.setdefault(e.name[:40], []).append(e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total)
    print("   kernels:", {k: round(sum(v) / len(v) / 1e3, 3) for k, v in ks.items()}, flush=True)
    nnz = U.batch_nnz(jag, m)
    tf = 4 * 128 * 4 * nnz / (res["fwd"] / 1e3) / 1e12
    tb = 10 * 128 * 4 * nnz / (res["bwd"] / 1e3) / 1e12
    print(f"B={B} rab={rab} K1={K1} K2={K2}: fwd {res['fwd']:.3f} ms ({tf:.0f} TF/s)  bwd {res['bwd']:.3f} ms ({tb:.0f} TF/s)",
          flush=True)


if __name__ == "__main__":
    if os.environ.get("ATTN_TIME_SPLIT"):   # rab cost split: position table only / time buckets only
        run(rab="pos")
        run(rab="ts")
    run(rab=True)
    run(rab=False)
    run(rab=False, K1=16383, K2=0, B=4)
    if os.environ.get("ATTN_TIME_CAUSAL_RAB"):   # full causal with rab (cfg2's mask at 16k)
        run(rab=True, K1=16383, K2=0, B=4)
