import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    # UH_TEST_LIB=libuhstu_checked.so runs the suite against a variant build of the library
    # (tools/build_variant.py; the checked build traps on any device-side range violation)
    lib = os.environ.get("UH_TEST_LIB")
    if lib:
        from paper_2602_16986_b200 import uhstu as U
        U.LIB_PATH = os.path.join(ROOT, "paper_2602_16986_b200", "lib", lib)
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU; parity tests through the C-ABI")
    config.addinivalue_line("markers", "slow: long CPU/GPU runs (full-size configs)")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)
