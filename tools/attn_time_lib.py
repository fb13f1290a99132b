"""attn_time.run with an alternative library build (experiments).  usage: attn_time_lib.py <lib.so> B rab"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
from paper_2602_16986_b200 import uhstu as U  # noqa: E402

U.LIB_PATH = os.path.abspath(sys.argv[1])
from attn_time import run  # noqa: E402

run(B=int(sys.argv[2]), rab=bool(int(sys.argv[3])))
