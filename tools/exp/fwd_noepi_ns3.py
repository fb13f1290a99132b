import runpy, os
h = os.path.dirname(os.path.abspath(__file__))
PATCHES = runpy.run_path(os.path.join(h, "fwd_noepi.py"))["PATCHES"] + runpy.run_path(os.path.join(h, "fwd_ns3.py"))["PATCHES"]
