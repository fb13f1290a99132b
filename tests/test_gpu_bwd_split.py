"""The two-kernel attention backward (UH_ATTN_BWD=split: query-major dQ kernel + key-major
dK/dV kernel) stays parity-green next to the default fused kernel.  The variable is read once
per process, so the check runs in a subprocess."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys
sys.path[:0] = [{root!r}, {tests!r}, {oracle!r}]
from test_gpu_parity import AttnCase, RAGGED, check_bwd
from paper_2602_16986_b200 import synth
from paper_2602_16986_b200 import uhstu as U
for K1, K2 in [(16, 2), (127, 129), (synth.WINDOW_FULL, 0)]:
    check_bwd(AttnCase(RAGGED + [300], H=2, dh=128, K1=K1, K2=K2, N=300.0, P=40, seed=6), U.BF16)
print("split ok")
"""


def test_split_backward_parity():
    code = SCRIPT.format(root=ROOT, tests=os.path.join(ROOT, "tests"), oracle=os.path.join(ROOT, "oracle"))
    env = dict(os.environ, UH_ATTN_BWD="split")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "split ok" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]
