"""One attention fwd+bwd at cfg3 shape (B sequences) for ncu.  usage: prof_attn.py B rab(0/1)"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
from attn_time import run  # noqa: E402

if __name__ == "__main__":
    B = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    rab = bool(int(sys.argv[2])) if len(sys.argv) > 2 else False
    run(B=B, rab=rab, steps=1)
