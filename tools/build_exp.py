"""Experiment builds (not product code): copy csrc/ to a scratch directory, apply literal
(old -> new) patches from a spec module, and link lib/libuhstu_<name>.so.
usage: build_exp.py NAME SPEC.py   (SPEC defines PATCHES = [(file, old, new), ...])"""
import concurrent.futures as cf
import glob
import os
import runpy
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "paper_2602_16986_b200"))
import build as B  # noqa: E402

name, spec = sys.argv[1], sys.argv[2]
spec_ns = runpy.run_path(spec)
patches = spec_ns["PATCHES"]            # (file, old, new); old None: replace the whole file with new
extra = spec_ns.get("FLAGS", [])
tmp = tempfile.mkdtemp(prefix="uhexp_")
src = os.path.join(tmp, "pkg", "csrc")   # internal.h includes ../../include/uhstu.h
shutil.copytree(B.CSRC, src)
shutil.copytree(os.path.join(ROOT, "include"), os.path.join(tmp, "include"))
for f, old, new in patches:
    p = os.path.join(src, f)
    if old is None:
        open(p, "w").write(new)
        continue
    s = open(p).read()
    assert old in s, (f, old[:80])
    open(p, "w").write(s.replace(old, new))
obj_dir = os.path.join(tmp, "obj")
os.makedirs(obj_dir)
flags = [fl if not fl.startswith("-I" + B.CSRC) else "-I" + src for fl in B.FLAGS] + extra


def comp(cu):
    obj = os.path.join(obj_dir, os.path.basename(cu).replace(".cu", ".o"))
    r = subprocess.run([B.NVCC, *B.ARCH, *flags, "-c", cu, "-o", obj], capture_output=True, text=True)
    if r.returncode:
        raise RuntimeError(r.stderr)
    for ln in r.stderr.splitlines():          # -Xptxas -warn-spills
        if "spill" in ln.lower() or "stack frame" in ln.lower():
            print(os.path.basename(cu), ln.strip())
    return obj


with cf.ThreadPoolExecutor(8) as ex:
    objs = list(ex.map(comp, sorted(glob.glob(os.path.join(src, "*.cu")))))
lib = os.path.join(os.path.dirname(B.LIB), f"libuhstu_{name}.so")
r = subprocess.run([B.NVCC, *B.ARCH, "-shared", "-o", lib, *objs, "-cudart", "shared", "-Xcompiler", "-fPIC"],
                   capture_output=True, text=True)
if r.returncode:
    raise RuntimeError(r.stderr)
shutil.rmtree(tmp)
print(lib)
