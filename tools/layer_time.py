"""Time one cfg3 layer forward (training, saving the remat set) and backward through the C ABI
(CUDA events); UH_LIB=libuhstu_<name>.so selects an experiment build."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2602_16986_b200 import synth  # noqa: E402
from paper_2602_16986_b200 import uhstu as U  # noqa: E402
if os.environ.get("UH_LIB"):
    U.LIB_PATH = os.path.join(ROOT, "paper_2602_16986_b200", "lib", os.environ["UH_LIB"])


def t(fn, it=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(it):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / it


cfg = synth.config("cfg3")
p = synth.layer_params(cfg.d, cfg.seed)
pos, ts = synth.rab_tables(cfg)
tt = synth.timestamps(cfg.seed, cfg.lengths)
f = lambda a: torch.from_numpy(a).cuda()
b = lambda a: torch.from_numpy(a).to("cuda", torch.bfloat16)
prm = U.Params(f(p["ln1_w"]), f(p["ln1_b"]), b(p["w1"]), f(p["ln2_w"]), f(p["ln2_b"]), b(p["w2"]), f(p["b1"]), f(p["b2"]))
attn = U.Attn(cfg.H, cfg.dh, 1.0, float(cfg.N), f(pos), f(ts), f(tt))
jag = U.JaggedBatch(cfg.offsets())
m = U.mask(cfg.K1, cfg.K2)
X = torch.randn(cfg.T, cfg.d, device="cuda").to(torch.bfloat16)
D = torch.randn(cfg.T, cfg.d, device="cuda").to(torch.bfloat16)
out = torch.empty_like(X)
saved = U.alloc_saved(X)
wf = U._ws(U.layer_workspace_bytes(jag, m, prm, attn, U.BF16, False), "cuda")
wb = U._ws(U.layer_workspace_bytes(jag, m, prm, attn, U.BF16, True), "cuda")
dx = torch.empty_like(X)
fwd = lambda: U.layer_fwd(jag, m, prm, attn, X, out=out, ws=wf, saved=saved)
fwd()
bwd = lambda: U.layer_bwd(jag, m, prm, attn, X, saved, D, dx=dx, ws=wb)
ms_f, ms_b = t(fwd), t(bwd)
print(f"cfg3 layer: fwd {ms_f:.3f} ms  bwd {ms_b:.3f} ms  step {ms_f + ms_b:.3f} ms", flush=True)
