"""NEXT-3 LBSL timing on one B200: host selection per rank-step (b = 32 users, the paper's
regime of long histories) and the device gather of the kept rows (HBM roofline: 2 bytes
moved per kept element byte, read + write)."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_16986_b200 import lbsl as NL
from paper_2602_16986_b200 import uhstu as U

rng = np.random.default_rng(0)
b, d = 32, 512
rt = NL.LBSL(NL.LbslConfig(T_warm=3, T_recal=10, gamma=1.7, ell_sl=1024, seed=1))
B = [int(min(16384, 512 * (1 + rng.pareto(1.5)))) for _ in range(b)]
for _ in range(5):
    rt.select(B)
t0 = time.perf_counter()
n_sel = 2000
for _ in range(n_sel):
    dec, new = rt.select(B)
sel_us = (time.perf_counter() - t0) / n_sel * 1e6
t0 = time.perf_counter()
for _ in range(200):
    rows, off = U.lbsl_rows(np.concatenate([[0], np.cumsum(B)]), dec, new, 1, 0, rt.t)
rows_us = (time.perf_counter() - t0) / 200 * 1e6
# device gather at a large jagged batch: 2M tokens x 512 bf16 -> kept half
T = 2 * 1024 * 1024
x = torch.randn(T, d, device="cuda", dtype=torch.bfloat16)
idx = torch.sort(torch.randperm(T, device="cuda")[: T // 2]).values.to(torch.int32)
y = torch.empty(T // 2, d, device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    U.gather_rows(idx, x, out=y)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    U.gather_rows(idx, x, out=y)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
byts = (T // 2) * d * 2 * 2 + (T // 2) * 4
print(json.dumps({"select_us_per_rank_step": sel_us, "rows_us_per_rank_step": rows_us, "kept_tokens": int(sum(new)),
                  "gather_ms": ms, "gather_GBps": byts / ms / 1e6, "gather_bytes": byts}))
