"""Timeline of CTA 0 of the forward kernel (trace build): per tile, when the MMA warp got
K/V, when it got P, and when epilogue warp 4 waited for / got S and finished P."""
import ctypes, os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2602_16986_b200 import uhstu as U
U.LIB_PATH = os.path.join(ROOT, "paper_2602_16986_b200", "lib", "libuhstu_trace_item.so")
L = U.lib()
buf = torch.zeros(8192, dtype=torch.int64, device="cuda")
L.uh_trace_set.argtypes = [ctypes.c_void_p]
print("set", L.uh_trace_set(ctypes.c_void_p(buf.data_ptr())))
sys.path.insert(0, os.path.join(ROOT, "tools"))
from attn_time import run
run(B=16, rab=bool(int(sys.argv[1])) if len(sys.argv) > 1 else False, steps=1)
t = buf.view(8, 1024).cpu().numpy()
t0 = t[t > 0].min()
names = ["S_issue", "PV_issue", "w4_wait_s", "w4_got_s", "w4_computed", "w4_arrived", "w4_oempty", "w4_setup"]
for j in range(400, 440):
    row = [(t[e, j] - t0) if t[e, j] > 0 else -1 for e in range(8)]
    print(j, " ".join(f"{n}={v:8d}" for n, v in zip(names, row)))
for e, n in enumerate(names):
    x = np.sort(t[e][t[e] > 0])
    if len(x) > 10:
        print(f"{n}: median interval {np.median(np.diff(x)):.0f} cycles")
