"""Regenerate profiles/r02_summary.md from the committed round-2 evidence (no GPU needed):
the bench line, the launch list of one layer step, the ncu --set full summaries of every kernel
(DRAM bytes against each kernel's algorithmic bytes, tensor-pipe activity against its FLOPs),
the cfg5 lines and the checked-build test log."""
import csv
import json
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
P = os.path.join(ROOT, "profiles")
T, D = 262144, 512                     # cfg3 tokens per GPU, model width
MB = 1e6

# (pattern, label, algorithmic bytes or None, algorithmic flops or None) per launch at cfg3
KERNELS = [
    (r"ln_fwd_k", "F1 LayerNorm", 2 * T * D * 2 + 8 * T, None),
    (r"gemm_bf16_sm100<256, 0, 1, 1, 1", "F2 f1 + SiLU / B3 remat f1 (+ silu')", None, 2 * T * D * 4 * D),
    (r"build_schedule_k", "F0 tile schedule", None, None),
    (r"rab_ext_k", "rab: extended position table", None, None),
    (r"attn_fwd_sm100", "F3-F5 attention forward", None, 4 * 128 * 4 * 18226624 * 16),
    (r"gated_fwd_k", "F6 gated norm", 3 * T * D * 2 + 8 * T, None),
    (r"gemm_bf16_sm100<256, 0, 1, 0, 1", "F7 f2 + residual", None, 2 * T * D * D),
    (r"ln_apply_k", "B3 x^ from saved statistics", 2 * T * D * 2 + 8 * T, None),
    (r"gemm_bf16_sm100<256, 0, 0, 0, 1", "B1 dY", None, 2 * T * D * D),
    (r"gated_bwd", "B2 gated-norm backward", 7 * T * D * 2, None),
    (r"gemm_bf16_sm100<256, 1, 1, 2, 2", "B1 dW2 / B5 dW1 (split-K, fused bias sums)", None, None),
    (r"attn_bwd_fused_sm100", "B4 attention backward (fused dK, dV, dQ)", None, 10 * 128 * 4 * 18226624 * 16),
    (r"dq_finish_k", "B4 dQ finish", T * D * 4 + 2 * T * D * 2, None),
    (r"gemm_bf16_sm100<256, 0, 0, 0, 2", "B5 dx^", None, 2 * T * 4 * D * D),
    (r"ln_bwd", "B6 LayerNorm backward + residual", 4 * T * D * 2, None),
]


def label(name):
    for pat, lab, b, f in KERNELS:
        if re.search(pat, name):
            return lab, b, f
    return "?", None, None


def main():
    out = ["# Round 2 profile summary (cfg3: 16 x 16384 tokens, 4 x 128 heads, SLA 1024 + 128 global, "
           "rab on with P = 16384, NB = 32)", ""]
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"hbm_gbs": 6543.1, "bf16_tflops": 1700.9}
    b = json.load(open(os.path.join(P, "r02_bench.json")))
    at, rf = b["attn"], b["roofline"]
    out += ["## Bench line (`python bench.py --steps 20 --warmup 5`, one B200): `r02_bench.json`", ""]
    out += [f"Layer step {b['ms_per_step']:.2f} ms = {b['value'] / 1e6:.1f} M tokens/s. Attention fwd "
            f"{at['fwd_ms']:.3f} ms / bwd {at['bwd_ms']:.3f} ms = {at['effective_tflops']:.0f} TFLOP/s effective "
            f"({100 * at['frac_of_measured_bf16_burst']:.1f}% of the measured bf16 burst). Roofline (attention "
            f"backward): {rf['achieved']:.0f} / {rf['peak']:.0f} TFLOP/s = {rf['frac']:.3f}. e2e "
            f"{b['e2e']['value'] / 1e6:.1f} M tokens/s; clocks {b['clocks']['sm_mhz']} MHz {b['clocks']['reasons']}.", ""]
    for n in (2, 4, 8):
        f = os.path.join(P, f"r02_bench_{n}gpu.json")
        if os.path.exists(f):
            d = json.loads(open(f).read().strip().splitlines()[-1])
            out.append(f"{n} GPUs (`r02_bench_{n}gpu.json`, self-launched `bench.py --gpus {n}`): "
                       f"{d['value'] / 1e6:.1f} M tokens/s at {d['ms_per_step']:.2f} ms per step "
                       f"({100 * d['value'] / (n * b['value']):.0f}% of {n} x one GPU); NCCL {d.get('nccl')}.")
    out.append("")
    lf = os.path.join(P, "r02_bench_launches.csv")
    if os.path.exists(lf):
        rows = [r for r in csv.reader(open(lf)) if len(r) > 10]
        h = rows[0]
        ki, vi = h.index("Kernel Name"), h.index("Metric Value")
        agg = {}
        for r in rows[1:]:
            nm = r[ki]
            lab = label(nm)[0]
            if lab == "?":   # not one of the library's kernels (torch fills / copies of the harness)
                lab = "other: `" + re.sub(r"\(.*", "", nm).replace("void ", "")[:48] + "`"

            agg.setdefault(lab, []).append(float(r[vi].replace(",", "")) / 1e3)
        out += ["## Launch list (`ncu --metrics gpu__time_duration.sum --clock-control none`, cold-cache, serialised): "
                "`r02_bench_launches.csv`", "",
                "Mean duration per launch over the bench run's launches (the attention-alone timing calls included).", "",
                "| step | launches | us per launch |", "|---|---|---|"]
        for lab, v in agg.items():
            out.append(f"| {lab} | {len(v)} | {sum(v) / len(v):.1f} |")
        out.append("")
    nf = os.path.join(P, "r02_ncu_layer_cfg3.json")
    if os.path.exists(nf):
        ks = json.load(open(nf))["kernels"]
        out += ["## Every kernel of one layer step, `ncu --set full`: `r02_ncu_layer_cfg3.json`", "",
                "HBM kernels: achieved DRAM GB/s against the measured copy peak "
                f"({peaks['hbm_gbs']:.0f} GB/s) and DRAM bytes against the algorithmic bytes; tensor kernels: "
                "tensor-pipe activity and algorithmic TFLOP/s against the measured bf16 burst "
                f"({peaks['bf16_tflops']:.0f} TFLOP/s).", "",
                "| step | kernel | us | DRAM GB | algorithmic GB | DRAM GB/s | frac of copy peak | tensor pipe % | "
                "TFLOP/s | frac of bf16 burst |", "|---|---|---|---|---|---|---|---|---|---|"]
        for k in ks:
            lab, ab, af = label(k["full_name"])
            if lab == "?":
                continue
            if "dW2 / B5 dW1" in lab:   # same instantiation: dW2 (K = T, N = d) is the short one
                af = 2 * T * D * D if k.get("time_ms", 0) < 0.25 else 2 * T * D * 4 * D
            t = k.get("time_ms", 0) * 1e3
            dram = (k.get("dram_read_bytes", 0) + k.get("dram_write_bytes", 0)) / 1e9
            gbs = k.get("dram_gbs", 0)
            tf = af / (t * 1e-6) / 1e12 if af and t else None
            out.append(f"| {lab} | `{k['kernel'][:40]}` | {t:.1f} | {dram:.3f} | "
                       f"{ab / 1e9:.3f} | " if ab else f"| {lab} | `{k['kernel'][:40]}` | {t:.1f} | {dram:.3f} | - | ")
            out[-1] += (f"{gbs:.0f} | {gbs / peaks['hbm_gbs']:.2f} | " if ab else f"{gbs:.0f} | - | ")
            out[-1] += f"{k.get('tensor_pipe_active_pct', 0):.1f} | "
            out[-1] += (f"{tf:.0f} | {tf / peaks['bf16_tflops']:.2f} |" if tf else "- | - |")
        out.append("")
    for L in (4096, 16384, 65536):
        f = os.path.join(P, f"r02_cfg5_L{L}.json")
        if os.path.exists(f):
            d = json.loads(open(f).read().strip().splitlines()[-1])
            out.append(f"cfg5 L = {L} (`r02_cfg5_L{L}.json`): {d['value'] / 1e6:.2f} M input tokens/s, "
                       f"{d['config']['workload']}, HBM {d['config'].get('hbm_used_gb', 0):.0f} GB.")
    out.append("")
    mf = os.path.join(P, "r02_mot_bench.json")
    if os.path.exists(mf):
        d = json.loads(open(mf).read().strip().splitlines()[-1])
        out += ["## NEXT-4 Mixture of Transducers (`bench.py --config mot`): `r02_mot_bench.json`", "",
                f"{d['value'] / 1e6:.1f} M input tokens/s at {d['ms_per_step']:.2f} ms per training step; "
                f"{d['config']['workload']}.", ""]
    af = os.path.join(P, "r02_attn_time.log")
    if os.path.exists(af):
        out += ["## Attention kernels alone (`tools/attn_time.py`, CUDA events): `r02_attn_time.log`", "", "```"]
        out += [ln.strip() for ln in open(af) if ln.strip()] + ["```", ""]
    ff = os.path.join(P, "r02_fp8_time.log")
    if os.path.exists(ff):
        out += ["## Projections, bf16 and FP8 (NEXT-2): `r02_fp8_time.log`, `r02_ncu_gemm_cfg3.json`", "", "```"]
        out += [ln.rstrip() for ln in open(ff) if ln.strip() and not ln.startswith("#")] + ["```", ""]
    gf = os.path.join(P, "r02_ncu_gemm_cfg3.json")
    if os.path.exists(gf):
        out += ["| GEMM | us | tensor pipe % | L1/smem % | issue % | SM GHz |", "|---|---|---|---|---|---|"]
        for k in json.load(open(gf))["kernels"]:
            out.append(f"| {k['gemm']} | {k['time_us']:.0f} | {k['tensor_pipe_active_pct']:.1f} | "
                       f"{k['l1tex_throughput_pct']:.1f} | {k['issue_active_pct']:.1f} | {k['sm_clock_ghz']:.2f} |")
        out.append("")
    cf = os.path.join(P, "r02_checked_tests.log")
    if os.path.exists(cf):
        last = [ln for ln in open(cf).read().splitlines() if ln.strip()][-1]
        out += ["## Checked build (`-DUH_CHECKED=1`: device-side range checks trap on violation)", "",
                f"`UH_TEST_LIB=libuhstu_checked.so pytest tests -m gpu`: {last} (`r02_checked_tests.log`). "
                "compute-sanitizer is closed on the GPU pool (`r02_sanitizer_refused.txt`).", ""]
    open(os.path.join(P, "r02_summary.md"), "w").write("\n".join(out) + "\n")
    print("\n".join(out))


if __name__ == "__main__":
    main()
