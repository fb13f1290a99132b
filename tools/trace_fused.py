"""Timeline of CTA 0 of the fused attention backward (build: tools/build_variant.py trace3 -DUH_TRACE=3).
usage: trace_fused.py [first_step] [count] [rab 0/1]"""
import ctypes, os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2602_16986_b200 import synth
from paper_2602_16986_b200 import uhstu as U
U.LIB_PATH = os.path.join(ROOT, "paper_2602_16986_b200", "lib", "libuhstu_trace3.so")
L = U.lib()
cfg = synth.config("cfg3")
lengths = [16384] * 16
jag = U.JaggedBatch.from_lengths(lengths)
T, d = jag.T, cfg.d
g = torch.Generator().manual_seed(0)
buf = (torch.randn(T, 4 * d, generator=g) * (4.0 / 128) ** 0.25).to("cuda", torch.bfloat16)
q, k, v = buf[:, 2 * d:3 * d], buf[:, 3 * d:], buf[:, d:2 * d]
dA = torch.randn(T, d, generator=g).to("cuda", torch.bfloat16)
pos, ts = synth.rab_tables(cfg)
t = synth.timestamps(cfg.seed, lengths)
rab = int(sys.argv[3]) if len(sys.argv) > 3 else 1
attn = U.Attn(4, 128, 1.0, float(cfg.N), torch.from_numpy(pos).cuda() if rab else None,
              torch.from_numpy(ts).cuda() if rab else None, torch.from_numpy(t).cuda() if rab else None)
m = U.mask(1024, 128)
gb = torch.empty(T, 3 * d, dtype=torch.bfloat16, device="cuda")
wb = U._ws(U.attn_workspace_bytes(jag, m, attn, U.BF16, True), "cuda")
tb = torch.zeros(8192, dtype=torch.int64, device="cuda")
L.uh_trace_set_bwd.argtypes = [ctypes.c_void_p]
for _ in range(2):
    U.attn_bwd(jag, m, attn, q, k, v, dA, gb[:, :d], gb[:, d:2 * d], gb[:, 2 * d:], ws=wb)
L.uh_trace_set_bwd(ctypes.c_void_p(tb.data_ptr()))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
U.attn_bwd(jag, m, attn, q, k, v, dA, gb[:, :d], gb[:, d:2 * d], gb[:, 2 * d:], ws=wb)
e1.record()
torch.cuda.synchronize()
print("bwd ms (traced)", e0.elapsed_time(e1))
tr = tb.view(8, 1024).cpu().numpy()
t0 = tr[tr > 0].min()
names = ["A_issue", "BC_issue", "E1a_sfull", "E1a_pfull", "E1b_sfull", "E2_dqfull", "E2_dsfree", "QA_load"]
first = int(sys.argv[1]) if len(sys.argv) > 1 else 300
cnt = int(sys.argv[2]) if len(sys.argv) > 2 else 40
for j in range(first, first + cnt):
    row = [(tr[e, j] - t0) if tr[e, j] > 0 else -1 for e in range(8)]
    print(j, " ".join(f"{n}={v:9d}" for n, v in zip(names, row)))
import numpy as np
for e, n in enumerate(names):
    x = tr[e][tr[e] > 0]
    x = np.sort(x)
    if len(x) > 10:
        print(f"{n}: median step interval {np.median(np.diff(x)):.0f} cycles")
