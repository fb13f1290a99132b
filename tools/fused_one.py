"""One bf16 attention backward call (the ragged test's shapes) for compute-sanitizer runs."""
import sys
sys.path.insert(0, "tests")
sys.path.insert(0, ".")
sys.path.insert(0, "oracle")
import torch
from test_gpu_parity import AttnCase, RAGGED, run_bwd, oracle_bwd
from gpu_util import rel_inf
from paper_2602_16986_b200 import uhstu as U

K1, K2 = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (16, 2)
case = AttnCase(RAGGED + [300], H=2, dh=128, K1=K1, K2=K2, N=300.0, P=40, seed=6)
got = run_bwd(case, U.BF16)
ref = oracle_bwd(case)
for n, g, r in zip(["dQ", "dK", "dV", "dpos", "dts"], got, ref):
    if r is not None:
        print(n, rel_inf(g, r))
