import os, runpy
PATCHES = runpy.run_path(os.path.join(os.path.dirname(os.path.abspath(__file__)), "fwd_old.py"))["PATCHES"]
FLAGS = ["-DUH_EXP=1"]
