"""Build a variant of libuhstu.so with extra nvcc defines (trace / experiment builds).
usage: build_variant.py NAME -DFOO=1 ...   ->  paper_2602_16986_b200/lib/libuhstu_NAME.so"""
import concurrent.futures as cf
import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "paper_2602_16986_b200"))
import build as B  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
obj_dir = os.path.join(os.path.dirname(B.LIB), "obj_" + name)
os.makedirs(obj_dir, exist_ok=True)
srcs = sorted(glob.glob(os.path.join(B.CSRC, "*.cu")))


def comp(src):
    obj = os.path.join(obj_dir, os.path.basename(src).replace(".cu", ".o"))
    r = subprocess.run([B.NVCC, *B.ARCH, *B.FLAGS, *defs, "-c", src, "-o", obj], capture_output=True, text=True)
    if r.returncode:
        raise RuntimeError(r.stderr)
    return obj


with cf.ThreadPoolExecutor(8) as ex:
    objs = list(ex.map(comp, srcs))
lib = os.path.join(os.path.dirname(B.LIB), f"libuhstu_{name}.so")
r = subprocess.run([B.NVCC, *B.ARCH, "-shared", "-o", lib, *objs, "-cudart", "shared", "-Xcompiler", "-fPIC"],
                   capture_output=True, text=True)
if r.returncode:
    raise RuntimeError(r.stderr)
print(lib)
