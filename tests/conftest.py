import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path)")
    config.addinivalue_line("markers", "slow: long-running (full-size or exhaustive sweeps)")
    # The native libraries are build products (git-ignored). In a fresh
    # checkout, build them once before collecting (nvcc cross-compiles
    # sm_100a without a GPU; a few minutes).
    needed = [os.path.join(ROOT, "paper_2412_00408_b200", "libquake_b200.so"),
              os.path.join(ROOT, "oracle", "liboracle.so")]
    if not all(os.path.exists(f) for f in needed):
        import __graft_entry__
        __graft_entry__.build()


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)
