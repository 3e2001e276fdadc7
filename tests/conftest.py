import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run under gpurun)")


def pytest_collection_modifyitems(config, items):
    # GPU tests run only when CUDA is present; never silently pass without it.
    try:
        import torch

        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device (run with gpurun)")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


def pytest_sessionstart(session):
    # libtlk.so is built in-tree; build it here if the checkout has none yet
    lib = os.path.join(ROOT, "paper_2410_22254_b200", "_lib", "libtlk.so")
    if not os.path.exists(lib):
        from paper_2410_22254_b200.build import build

        build()
