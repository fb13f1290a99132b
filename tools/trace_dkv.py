"""Timeline of CTA 0 of the dK/dV kernel (trace build)."""
import ctypes, os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2602_16986_b200 import uhstu as U
U.LIB_PATH = os.path.join(ROOT, "paper_2602_16986_b200", "lib", "libuhstu_trace.so")
L = U.lib()
buf = torch.zeros(8192, dtype=torch.int64, device="cuda")
L.uh_trace_set_bwd.argtypes = [ctypes.c_void_p]
print("set", L.uh_trace_set_bwd(ctypes.c_void_p(buf.data_ptr())))
sys.path.insert(0, os.path.join(ROOT, "tools"))
from attn_time import run
run(B=int(sys.argv[2]) if len(sys.argv) > 2 else 2, rab=bool(int(sys.argv[1])) if len(sys.argv) > 1 else False, steps=1)
t = buf.view(8, 1024).cpu().numpy()
t0 = t[t > 0].min()
names = ["w1_beg", "w1_lastS", "w3_beg", "w3_last", "ep_accfull", "ep_accempty", "ep_stored", "x"]
for j in range(int(sys.argv[3]) if len(sys.argv) > 3 else 0, (int(sys.argv[3]) if len(sys.argv) > 3 else 0) + 24):
    row = [(t[e, j] - t0) if t[e, j] > 0 else -1 for e in range(8)]
    print(j, " ".join(f"{n}={v:8d}" for n, v in zip(names, row)))
tt = t[t > 0]
print("span cycles", tt.max() - tt.min())
