"""bench.py — throughput of the ULTRA-HSTU hot path on B200 (BASELINE.json metric:
"HSTU attn effective TFLOP/s & tokens/s at L=16k vs bf16 peak, 1/2/4/8 B200").

A step = one pass of the whole hot path over one batch of synthetic
input: the jagged schedule, LN, f1+SiLU, SLA attention, gated norm, f2+residual
(forward), then the rematerialising backward (LN apply, f1 remat, dY/dW2, gated-norm
backward, attention backward, dW1/dx^, LN backward) and — for N > 1 — the NCCL
all-reduce of the layer's fp32 weight-gradient bucket.  Each rank runs the cfg3
shape (16 x 16384 tokens, 4 heads x 128, window 1024 + 128 global, rab on), so
per-GPU work is fixed as N grows ("scaling": "weak"); the global batch is sharded by
the LPT token-balanced partitioner (uh_partition_lpt).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config cfg3|cfg2|cfg4]

Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "HSTU attn effective TFLOP/s & tokens/s at L=16k vs bf16 peak, 1/2/4/8 B200"


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return {"bf16_tflops": d["bf16_tflops"], "bf16_tflops_sustained": d.get("bf16_tflops_sustained"),
                "hbm_gbs": d["hbm_gbs"], "source": "measured"}
    except Exception:
        return {"bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "hbm_gbs": 6650.0, "source": "fallback"}


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi sampled every 200 ms during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, index: int):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={index}", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                       "-lms", "50"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        self.f.flush()
        self.f.seek(0)
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.f.read().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = max(mx, float(parts[2]))
            except ValueError:
                continue
            for n, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        os.unlink(self.f.name)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------- workload
def setup_workload(cfg_name: str, world: int, rank: int, device):
    import torch

    from paper_2602_16986_b200 import synth
    from paper_2602_16986_b200 import uhstu as U

    gcfg = synth.config(cfg_name, world=world)
    m = U.mask(gcfg.K1, gcfg.K2)
    owner, cost = U.partition_lpt(gcfg.lengths, world, m, gcfg.d, gcfg.H)
    ids = [i for i in range(len(gcfg.lengths)) if owner[i] == rank]
    lengths = [gcfg.lengths[i] for i in ids]
    x, dout = synth.layer_inputs(gcfg, ids=ids, lengths=lengths)
    t = synth.timestamps(gcfg.seed, lengths, ids=ids)
    pos, ts = synth.rab_tables(gcfg)
    p = synth.layer_params(gcfg.d, gcfg.seed)
    f = lambda a: torch.from_numpy(a).to(device)
    b = lambda a: torch.from_numpy(a).to(device, torch.bfloat16)
    prm = U.Params(f(p["ln1_w"]), f(p["ln1_b"]), b(p["w1"]), f(p["ln2_w"]), f(p["ln2_b"]), b(p["w2"]), f(p["b1"]),
                   f(p["b2"]))
    off = np.zeros(len(lengths) + 1, np.int32)
    off[1:] = np.cumsum(lengths)
    jag = U.JaggedBatch(off, device)
    attn = U.Attn(gcfg.H, gcfg.dh, gcfg.alpha, float(gcfg.N), f(pos), f(ts), f(t))
    return dict(cfg=gcfg, m=m, jag=jag, attn=attn, prm=prm, x_host=x, dout_host=dout, t_host=t, lengths=lengths,
                rank_cost=cost, owner=owner)


# ----------------------------------------------------------------------------- our arm
def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    from paper_2602_16986_b200 import uhstu as U

    torch.cuda.set_device(local_rank)
    device = torch.device("cuda", local_rank)
    W = setup_workload(args.config, world, rank, device)
    cfg, m, jag, attn, prm = W["cfg"], W["m"], W["jag"], W["attn"], W["prm"]
    T, d = jag.T, cfg.d
    x = torch.from_numpy(W["x_host"]).to(device, torch.bfloat16)
    dout = torch.from_numpy(W["dout_host"]).to(device, torch.bfloat16)
    out = torch.empty_like(x)
    dx = torch.empty_like(x)
    saved = U.alloc_saved(x)
    from paper_2602_16986_b200 import dist as D
    bucket = D.GradBucket.for_layer(prm, attn, device)
    flat, gviews = bucket.flat, bucket.views
    ws_f = U._ws(U.layer_workspace_bytes(jag, m, prm, attn, U.BF16, False), device)
    ws_b = U._ws(U.layer_workspace_bytes(jag, m, prm, attn, U.BF16, True), device)

    def layer_fb(xx, dd, at):   # the layer's forward + rematerialising backward (grads into the bucket)
        U.layer_fwd(jag, m, prm, at, xx, out=out, ws=ws_f, saved=saved)
        U.layer_bwd(jag, m, prm, at, xx, saved, dd, grads=bucket.views, dx=dx, ws=ws_b)

    # The layer's ~20 launches are stream-ordered with no host synchronisation (F0 runs on the
    # device), so the forward + backward is captured once as a CUDA graph and replayed; the
    # gradient all-reduce stays outside the graph (NCCL, every N the same path).
    stack = None
    if cfg.n_layers > 1:   # cfg4: the L-layer stack, per-layer buckets all-reduced as each backward ends
        from paper_2602_16986_b200 import synth as _synth
        layers = []
        for li in range(cfg.n_layers):
            pl = _synth.layer_params(d, cfg.seed, layer=li)
            f = lambda a: torch.from_numpy(a).to(device)
            bb = lambda a: torch.from_numpy(a).to(device, torch.bfloat16)
            layers.append((U.Params(f(pl["ln1_w"]), f(pl["ln1_b"]), bb(pl["w1"]), f(pl["ln2_w"]), f(pl["ln2_b"]),
                                    bb(pl["w2"]), f(pl["b1"]), f(pl["b2"])), attn))
        stack = D.Stack(jag, m, layers, x)
        args.no_graph = True
        args.no_e2e = True
    graph, graph_launches = None, 0
    if not args.no_graph:
        cs0 = torch.cuda.Stream(device)
        cs0.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(cs0):
            layer_fb(x, dout, attn)
        torch.cuda.current_stream().wait_stream(cs0)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        lc0 = U.launch_count()
        with torch.cuda.graph(graph):
            layer_fb(x, dout, attn)
        graph_launches = U.launch_count() - lc0   # kernels recorded into the graph (one replay = one step)

    def step(xx, dd):   # one DP training step of the layer on this rank's shard (+ grad all-reduce)
        if stack is not None:
            _, _, hs = stack.step(xx, dd)
            for hd in hs:
                hd.wait()
            return
        if graph is not None and xx is x and dd is dout:
            graph.replay()
        else:
            layer_fb(xx, dd, attn)
        bucket.allreduce_()

    def barrier():
        if world > 1:
            dist.barrier()

    def timed(fn, K):
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(K):
            fn()
        e1.record()
        torch.cuda.synchronize()
        barrier()
        ms = e0.elapsed_time(e1)
        if world > 1:
            tt = torch.tensor([ms], device=device)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ms = float(tt.item())
        return ms

    for _ in range(args.warmup):
        step(x, dout)
    torch.cuda.synchronize()
    sampler = ClockSampler(local_rank) if rank == 0 else None
    l0 = U.launch_count()
    ms = timed(lambda: step(x, dout), args.steps)
    launches = U.launch_count() - l0 + (graph_launches * args.steps if graph is not None else 0)
    ms_step = ms / args.steps
    total_tokens = T * world if cfg.name == "cfg3" else sum(cfg.lengths)
    value = total_tokens / (ms_step / 1e3)

    # ---- attention alone (fwd, bwd) on the same batch, CUDA events on the launching stream
    ok_rows = torch.empty(T, 4 * d, dtype=torch.bfloat16, device=device)
    g = torch.Generator(device="cpu").manual_seed(7)
    sd = (4.0 / cfg.dh) ** 0.25
    ok_rows.copy_((torch.randn(T, 4 * d, generator=g) * sd).to(torch.bfloat16))
    q, k, v = ok_rows[:, 2 * d:3 * d], ok_rows[:, 3 * d:], ok_rows[:, d:2 * d]
    dA = torch.randn(T, d, generator=g).to(device, torch.bfloat16)
    A = torch.empty(T, d, dtype=torch.bfloat16, device=device)
    gbuf = torch.empty(T, 3 * d, dtype=torch.bfloat16, device=device)
    dq, dk, dv = gbuf[:, :d], gbuf[:, d:2 * d], gbuf[:, 2 * d:]
    dpos, dts = torch.zeros_like(attn.pos_bias), torch.zeros_like(attn.time_bias)
    wsa_f = U._ws(U.attn_workspace_bytes(jag, m, attn, U.BF16, False), device)
    wsa_b = U._ws(U.attn_workspace_bytes(jag, m, attn, U.BF16, True), device)
    fa = lambda: U.attn_fwd(jag, m, attn, q, k, v, out=A, ws=wsa_f)
    fb = lambda: U.attn_bwd(jag, m, attn, q, k, v, dA, dq, dk, dv, dpos, dts, ws=wsa_b)
    for _ in range(2):
        fa(); fb()
    fwd_ms = timed(fa, args.steps) / args.steps
    bwd_ms = timed(fb, args.steps) / args.steps
    clocks = sampler.stop() if sampler else None   # sampled across all timed regions
    nnz = U.batch_nnz(jag, m)
    fwd_flop = 4.0 * cfg.dh * cfg.H * nnz
    bwd_flop = 10.0 * cfg.dh * cfg.H * nnz
    peaks = load_peaks()
    attn_tflops = (fwd_flop + bwd_flop) / ((fwd_ms + bwd_ms) / 1e3) / 1e12

    # ---- e2e through the public API from pinned host buffers: every step copies its inputs
    # (x, dOut, timestamps) host -> device and reads the gradient bucket back.  Step i+1's
    # inputs are copied on a second stream into the other of two slots while step i computes.
    e2e = None
    if not args.no_e2e:
        from dataclasses import replace as _replace
        xh = torch.from_numpy(W["x_host"]).to(torch.bfloat16).pin_memory()
        dh_ = torch.from_numpy(W["dout_host"]).to(torch.bfloat16).pin_memory()
        th = torch.from_numpy(W["t_host"]).pin_memory()
        gh = torch.empty(flat.numel(), dtype=torch.float32).pin_memory()
        cs = torch.cuda.Stream(device)
        slots = []
        for _ in range(2):
            tsd = torch.empty_like(attn.timestamps)
            slots.append(dict(x=torch.empty_like(x), d=torch.empty_like(dout), ts=tsd,
                              attn=_replace(attn, timestamps=tsd), copied=torch.cuda.Event(), free=torch.cuda.Event()))

        def h2d(sl):
            with torch.cuda.stream(cs):
                cs.wait_event(sl["free"])
                sl["x"].copy_(xh, non_blocking=True)
                sl["d"].copy_(dh_, non_blocking=True)
                sl["ts"].copy_(th, non_blocking=True)
                sl["copied"].record(cs)

        def e2e_run(K):
            start = torch.cuda.Event()
            start.record()
            cs.wait_event(start)          # the copies belong to the timed region
            h2d(slots[0])
            for i in range(K):
                sl = slots[i % 2]
                if i + 1 < K:
                    h2d(slots[(i + 1) % 2])
                torch.cuda.current_stream().wait_event(sl["copied"])
                D.layer_step(jag, m, prm, sl["attn"], sl["x"], sl["d"], bucket, saved=saved, out=out, dx=dx,
                             ws_f=ws_f, ws_b=ws_b)
                sl["free"].record()
                gh.copy_(flat, non_blocking=True)

        e2e_run(2)
        e_ms = timed(lambda: e2e_run(args.steps), 1) / args.steps
        e2e = {"value": total_tokens / (e_ms / 1e3), "unit": "tokens/s", "ms_per_step": e_ms,
               "h2d_bytes_per_step": int(xh.numel() * 2 + dh_.numel() * 2 + th.numel() * 8),
               "d2h_bytes_per_step": int(gh.numel() * 4),
               "note": "inputs copied from pinned host memory every step; step i+1's copy overlaps step i"}

    if rank != 0:
        return None
    line = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": (f"{cfg.name}: ULTRA-HSTU layer fwd+bwd, {len(W['lengths'])} jagged seqs x L="
                                f"{max(W['lengths'])} per GPU ({T} tokens), 4 heads x 128, SLA window {cfg.K1} + "
                                f"{cfg.K2} global, rab (P={cfg.P}, NB={cfg.ts_len}), N={int(cfg.N)}")
                               if cfg.n_layers == 1 else
                               (f"{cfg.name}: {cfg.n_layers}-layer ULTRA-HSTU stack fwd+bwd, {len(W['lengths'])} jagged "
                                f"seqs (log-uniform 512..16384) = {T} tokens on rank 0, 4 heads x 128, SLA {cfg.K1} + "
                                f"{cfg.K2} global, rab, per-layer grad buckets all-reduced as each backward ends"),
                   "global_batch_tokens": total_tokens, "seq_len": max(W["lengths"]),
                   "parallelism": f"dp{world} (LPT token-balanced shards, NCCL all-reduce of the fp32 grad bucket)",
                   "l2": "inputs larger than L2 (x 268 MB, step working set ~8 GB)",
                   "launch": "CUDA graph replay of the layer fwd+bwd" if graph is not None else "eager launches"},
        "attn": {"fwd_ms": fwd_ms, "bwd_ms": bwd_ms, "nnz_pairs_per_head": nnz,
                 "effective_tflops": attn_tflops, "fwd_tflops": fwd_flop / (fwd_ms / 1e3) / 1e12,
                 "bwd_tflops": bwd_flop / (bwd_ms / 1e3) / 1e12,
                 "frac_of_measured_bf16_burst": attn_tflops / peaks["bf16_tflops"],
                 "frac_of_datasheet_2250": attn_tflops / 2250.0,
                 "flop_convention": "4*dh*H*nnz fwd + 10*dh*H*nnz bwd (unmasked pairs only)"},
        "roofline": roofline_bwd(bwd_flop, bwd_ms, peaks, cfg.name, T, d),
        "gpu_launches": launches, "gpu_launches_per_step": launches / args.steps,
        "clocks": clocks, "e2e": e2e,
    }
    if world > 1:
        line["nccl"] = {"nranks": world, "version": ".".join(map(str, torch.cuda.nccl.version())),
                        "NCCL_ALGO": os.environ.get("NCCL_ALGO", "auto (NCCL's choice)"),
                        "collective": "all_reduce(SUM) of the fp32 gradient bucket, once per step"}
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(cfg, budget_s=args.cpu_budget)
    return line


ROOFLINE_PROFILE = "r02_ncu_attn_bwd_cfg3.json"   # ncu --set full of one uh_attn_bwd call at cfg3


def roofline_bwd(bwd_flop: float, bwd_ms: float, peaks: dict, workload: str, T: int, d: int):
    """The dominant step, attention backward (B4, one uh_attn_bwd call: the fused key-major
    kernel attn_bwd_fused_sm100 plus the dQ finish kernel) against the measured bf16 burst peak
    (timed alone).  achieved = 10 d_h H nnz algorithmic FLOPs per launch / the CUDA-event time of
    the call; traffic = DRAM read + write bytes per launch of the call's kernels from the committed
    ncu --set full capture of the same workload (profiles/ROOFLINE_PROFILE)."""
    achieved = bwd_flop / (bwd_ms / 1e3) / 1e12
    traffic = None
    prof = os.path.join(ROOT, "profiles", ROOFLINE_PROFILE)
    if workload == "cfg3" and os.path.exists(prof):
        with open(prof) as f:
            pr = json.load(f)
        traffic = sum(k["dram_read_bytes"] + k["dram_write_bytes"] for k in pr["kernels"])
    algo_bytes = 7 * T * d * 2   # read Q, K, V, dA; write dQ, dK, dV (bf16 [T, d] each)
    return {"kernel": "attention backward (attn_bwd_fused_sm100 + dq_finish_k, one uh_attn_bwd call)",
            "bound": "tensor", "achieved": achieved, "peak": peaks["bf16_tflops"], "unit": "TFLOP/s",
            "frac": achieved / peaks["bf16_tflops"], "peak_source": peaks["source"] + " (burst: timed alone)",
            "algorithmic_flop_per_launch": bwd_flop, "traffic": traffic, "algorithmic_bytes_per_launch": algo_bytes,
            "traffic_note": f"DRAM bytes per launch (ncu --set full, profiles/{ROOFLINE_PROFILE}); the algorithmic "
                            f"minimum is 7 T d 2 = {algo_bytes / 1e9:.2f} GB (read Q, K, V, dA; write dQ, dK, dV); the "
                            "excess is the fp32 dQ accumulator (zeroed, reduced into in L2, read by the finish kernel)"}


# ----------------------------------------------------------------------------- cfg5: inference
def run_inference(args, rank, world, local_rank):
    """cfg5 / NEXT-1: forward-only 18-layer stack with attention truncation —
    6 SLA layers (window 1024 + 128 global) on the full sequences, then the latest 1024 tokens of
    each sequence through 12 full-causal layers (stack.forward_truncated).  Replicas only: every
    GPU runs its own batch, no collective.  value = input tokens of all GPUs per second."""
    import torch
    import torch.distributed as dist

    from paper_2602_16986_b200 import stack as S
    from paper_2602_16986_b200 import synth
    from paper_2602_16986_b200 import uhstu as U

    torch.cuda.set_device(local_rank)
    device = torch.device("cuda", local_rank)
    L, l_keep, n_sla, n_at = args.seq_len, 1024, 6, 12
    d = 512
    if args.tokens > 0:
        B = max(1, args.tokens // L)
    else:   # fill the GPU: x + two ping-pong outputs + one layer workspace (+ timestamps) per token
        probe = U.JaggedBatch.from_lengths([L], device)
        pw = torch.zeros(1, device=device)
        pb = lambda n: torch.zeros(n, device=device)
        prm0 = U.Params(pb(d), pb(d), torch.zeros(d, 4 * d, dtype=torch.bfloat16, device=device), pb(d), pb(d),
                        torch.zeros(d, d, dtype=torch.bfloat16, device=device), pb(4 * d), pb(d))
        a0 = U.Attn(4, 128, 1.0, float(L), pb(L), pb(32), torch.zeros(L, dtype=torch.int64, device=device))
        ws_tok = U.layer_workspace_bytes(probe, U.mask(1024, 128), prm0, a0, U.BF16, False) / L
        per_tok = ws_tok + 3 * d * 2 + 8
        free, _ = torch.cuda.mem_get_info(device)
        B = max(1, int(0.93 * free / per_tok) // L)
        del probe, pw, prm0, a0
    cfg = synth.Config("cfg5", [L] * B, H=4, dh=128, K1=1024, K2=128, N=L, seed=5 + rank)
    # x ~ N(0, 1) drawn on the device in 1M-row chunks (a GPU-filling batch is tens of GB)
    x = torch.empty(B * L, d, dtype=torch.bfloat16, device=device)
    gx = torch.Generator(device=device).manual_seed(cfg.seed)
    for r0 in range(0, B * L, 1 << 20):
        r1 = min(B * L, r0 + (1 << 20))
        x[r0:r1] = torch.randn(r1 - r0, d, generator=gx, device=device).to(torch.bfloat16)
    pos, ts = synth.rab_tables(cfg)
    t = torch.from_numpy(synth.timestamps(cfg.seed, cfg.lengths)).to(device)
    f = lambda a: torch.from_numpy(a).to(device)
    bb = lambda a: torch.from_numpy(a).to(device, torch.bfloat16)
    layers = []
    for li in range(n_sla + n_at):
        pl = synth.layer_params(d, cfg.seed, layer=li)
        prm = U.Params(f(pl["ln1_w"]), f(pl["ln1_b"]), bb(pl["w1"]), f(pl["ln2_w"]), f(pl["ln2_b"]), bb(pl["w2"]),
                       f(pl["b1"]), f(pl["b2"]))
        attn = U.Attn(cfg.H, cfg.dh, 1.0, float(L), f(pos), f(ts), t)
        m = U.mask(cfg.K1, cfg.K2) if li < n_sla else U.mask()
        layers.append(S.Layer(prm, attn, m))
    jag = U.JaggedBatch(cfg.offsets(), device)
    ws = U._ws(U.layer_workspace_bytes(jag, U.mask(1024, 128), layers[0].params, layers[0].attn, U.BF16, False),
               device)
    bufs = [torch.empty_like(x), torch.empty_like(x)]

    def step():
        S.forward_truncated(jag, x, layers, n_sla, l_keep, norm_n_truncated=float(l_keep), ws=ws, bufs=bufs)

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    sampler = ClockSampler(local_rank) if rank == 0 else None
    barrier()
    torch.cuda.synchronize()
    l0 = U.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        step()
    e1.record()
    torch.cuda.synchronize()
    barrier()
    ms = e0.elapsed_time(e1)
    if world > 1:
        tt = torch.tensor([ms], device=device)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    launches = U.launch_count() - l0
    clocks = sampler.stop() if sampler else None
    if rank != 0:
        return None
    ms_step = ms / args.steps
    tokens = B * L * world
    return {"metric": "HSTU inference tokens/s (cfg5: 6 SLA layers + truncation to 1024 + 12 full-causal layers)",
            "value": tokens / (ms_step / 1e3), "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": f"cfg5: {B} sequences x L={L} per GPU ({B * L} tokens), 4 heads x 128, "
                                   f"{n_sla} SLA layers (1024 + 128 global), latest {l_keep} tokens, {n_at} causal layers, "
                                   f"rab P={L}",
                       "hbm_used_gb": torch.cuda.max_memory_allocated(device) / 1e9,
                       "parallelism": f"replicas x{world} (no collective)", "seq_len": L},
            "gpu_launches": launches, "clocks": clocks,
            "e2e": None, "e2e_note": "inference inputs (x) stay resident; not measured for cfg5"}


def run_mot(args, rank, world, local_rank):
    """NEXT-4: one Mixture-of-Transducers training step per GPU — the paper's "10k
    C-seq and 3k E-seq" row: per user a 10240-token consumption sequence through a
    2-layer SLA transducer and a 3072-token engagement sequence through a 1-layer SLA transducer
    (window 1024 + 128 global, rab on), the last 64 positions of each sequence are the candidates,
    the fusion projects the concatenated [C, 2d] embeddings to d (readings R28-R30), then the
    whole backward (fusion, both stacks; fp32 buckets all-reduced over NCCL for N > 1).
    value = input tokens (both branches) of all GPUs per second."""
    import torch
    import torch.distributed as dist

    from paper_2602_16986_b200 import dist as D
    from paper_2602_16986_b200 import mot as GM
    from paper_2602_16986_b200 import synth
    from paper_2602_16986_b200 import uhstu as U

    torch.cuda.set_device(local_rank)
    device = torch.device("cuda", local_rank)
    B, n_cand, d, H = args.mot_users, 64, 512, 4
    spec = [("C-seq", 10240, 2), ("E-seq", 3072, 1)]
    f = lambda a: torch.from_numpy(a).to(device)
    bb = lambda a: torch.from_numpy(a).to(device, torch.bfloat16)
    stacks, xs = [], []
    for k, (name, L, n_layers) in enumerate(spec):
        cfg = synth.Config(f"mot-{name}", [L] * B, H=H, dh=128, K1=1024, K2=128, N=L, seed=31 + 7 * rank + k)
        m = U.mask(cfg.K1, cfg.K2)
        pos, ts = synth.rab_tables(cfg)
        t = f(synth.timestamps(cfg.seed, cfg.lengths))
        layers = []
        for li in range(n_layers):
            pl = synth.layer_params(d, cfg.seed, layer=li)
            prm = U.Params(f(pl["ln1_w"]), f(pl["ln1_b"]), bb(pl["w1"]), f(pl["ln2_w"]), f(pl["ln2_b"]),
                           bb(pl["w2"]), f(pl["b1"]), f(pl["b2"]))
            layers.append((prm, U.Attn(H, 128, 1.0, float(L), f(pos), f(ts), t)))
        x = torch.randn(B * L, d, generator=torch.Generator(device=device).manual_seed(cfg.seed), device=device)
        x = x.to(torch.bfloat16)
        xs.append(x)
        stacks.append(D.Stack(U.JaggedBatch(cfg.offsets(), device), m, layers, x))
    W, bias = synth.mot_params(d, len(spec), 41)
    mot = GM.MoT(stacks, n_cand, bb(W), f(bias))
    dE = torch.randn(B * n_cand, d, generator=torch.Generator(device=device).manual_seed(43 + rank),
                     device=device).to(torch.bfloat16)

    def step():
        mot.forward(xs)
        _, handles = mot.backward(xs, dE)
        for h in handles:
            h.wait()

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    sampler = ClockSampler(local_rank) if rank == 0 else None
    barrier()
    torch.cuda.synchronize()
    l0 = U.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        step()
    e1.record()
    torch.cuda.synchronize()
    barrier()
    ms = e0.elapsed_time(e1)
    if world > 1:
        tt = torch.tensor([ms], device=device)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    launches = U.launch_count() - l0
    clocks = sampler.stop() if sampler else None
    if rank != 0:
        return None
    ms_step = ms / args.steps
    tokens = B * sum(L for _, L, _ in spec) * world
    return {"metric": "MoT training tokens/s (NEXT-4: 10k C-seq 2 SLA layers + 3k E-seq 1 SLA layer + fusion, fwd+bwd)",
            "value": tokens / (ms_step / 1e3), "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": f"mot: {B} users per GPU; C-seq L=10240 x 2 layers, E-seq L=3072 x 1 layer, "
                                   f"d=512, 4 heads x 128, SLA 1024 + 128 global, rab P=L, {n_cand} candidates "
                                   f"per user, fusion [2d -> d]",
                       "parallelism": f"dp{world}", "inputs_exceed_l2": True},
            "gpu_launches": launches, "clocks": clocks,
            "e2e": None, "e2e_note": "inputs stay resident; not measured for the MoT workload"}


# ----------------------------------------------------------------------------- oracle arm
def oracle_sample(cfg, L: int):
    """The oracle (as it stands) on one length-L sequence of the workload: layer fwd+bwd."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O

    from paper_2602_16986_b200 import synth
    sub = synth.Config(cfg.name, [L], H=cfg.H, dh=cfg.dh, K1=cfg.K1, K2=cfg.K2, N=cfg.N, seed=cfg.seed,
                       pos_len=cfg.P, ts_len=cfg.ts_len)
    p = synth.layer_params(cfg.d, cfg.seed)
    x, dout = synth.layer_inputs(sub)
    pos, ts = synth.rab_tables(cfg)
    t = synth.timestamps(cfg.seed, [L])
    prm = O.LayerParams(**{k: np.asarray(v, np.float64) for k, v in p.items()})
    spec = O.AttnSpec(K1=O.FULL if cfg.K1 >= synth.WINDOW_FULL else cfg.K1, K2=cfg.K2, alpha=cfg.alpha, N=cfg.N,
                      pos_w=pos, ts_w=ts, timestamps=t)
    t0 = time.perf_counter()
    out, cache = O.layer_forward(x, sub.offsets(), prm, cfg.H, spec)
    O.layer_backward(dout, sub.offsets(), prm, cfg.H, spec, cache=cache)
    return time.perf_counter() - t0, O.num_threads()


def cpu_baseline(cfg, budget_s=20.0):
    L = 4096  # per-token attention work at L=4096 ~ L=16k under the 1024+128 window
    dt, cores = oracle_sample(cfg, L)
    return {"value": L / dt, "unit": "tokens/s", "cores": cores, "kind": "oracle",
            "sample": f"one {L}-token sequence of {cfg.name} (same dims/mask/rab), layer fwd+bwd, "
                      f"fp64 C pair loops (OpenMP) + numpy GEMMs; {dt:.1f} s"}


def run_reference(args, rank, world):
    if rank != 0:
        return None
    from paper_2602_16986_b200 import synth
    cfg = synth.config(args.config)
    L = 2048
    for _ in range(args.warmup):
        oracle_sample(cfg, 256)
    times = []
    cores = 1
    for _ in range(args.steps):
        dt, cores = oracle_sample(cfg, L)
        times.append(dt)
    ms = 1e3 * sum(times) / len(times)
    value = L / (ms / 1e3)
    return {"impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{cfg.name} (bounded sample: one {L}-token sequence per step)"},
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": cores, "kind": "oracle",
                             "sample": f"one {L}-token sequence of {cfg.name} per step, layer fwd+bwd"},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg3", choices=["cfg2", "cfg3", "cfg4", "cfg5", "mot"])
    ap.add_argument("--seq-len", type=int, default=16384, help="cfg5: sequence length (4096, 16384, 65536)")
    ap.add_argument("--tokens", type=int, default=4 * 1048576,
                    help="cfg5: tokens per GPU (0: as many as fill the GPU's free memory, BASELINE's cfg5)")
    ap.add_argument("--mot-users", type=int, default=16, help="mot: users per GPU")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="launch the step eagerly instead of replaying a CUDA graph")
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    args = ap.parse_args()
    warmup_requested = args.warmup
    if args.warmup < 3:   # the contract's minimum; the line reports the warm-up actually run
        args.warmup = 3
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # self-launch: one process per GPU through torch.distributed.run (same as the driver's torchrun)
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
        os.execv(sys.executable, cmd)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl != "reference" and world != args.gpus:
        sys.stderr.write(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}\n")
        sys.exit(2)
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    # stdout carries only the JSON line: native libraries (NCCL's version banner) write to
    # fd 1 from C, so point fd 1 at stderr and keep a private handle for the line
    out = os.fdopen(os.dup(1), "w")
    sys.stdout.flush()
    os.dup2(2, 1)
    if args.impl == "reference":
        line = run_reference(args, rank, world)
    else:
        if world > 1:
            import torch
            import torch.distributed as dist
            torch.cuda.set_device(local_rank)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        run = {"cfg5": run_inference, "mot": run_mot}.get(args.config, run_ours)
        line = run(args, rank, world, local_rank)
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
    if line is not None:
        if warmup_requested != args.warmup:
            line["warmup_requested"] = warmup_requested
        print(json.dumps(line), file=out, flush=True)


if __name__ == "__main__":
    main()
