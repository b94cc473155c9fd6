import importlib
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)

# The reference package (densefeed + densefeed_bindings), unmodified: installed into baseline/_ref with
# `pip install --no-index --no-build-isolation --no-deps --target baseline/_ref <copy of /root/reference/pkg>`
# (DESIGN.md §6); baseline/_ref travels to the GPU box with the repo snapshot.  In this container the
# read-only sources under /root/reference are an equivalent fallback.
REF_PATHS = [os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src", "/root/reference/pkg/bindings/src"]


def import_reference():
    """(densefeed, densefeed_bindings) from the unmodified reference.  Raises (never skips) when absent, so
    a test that drives the B200 step through the reference's seams cannot pass silently without it."""
    for p in REF_PATHS:
        if os.path.isdir(p) and p not in sys.path:
            sys.path.append(p)
    return importlib.import_module("densefeed"), importlib.import_module("densefeed_bindings")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")
    config.addinivalue_line("markers", "slow: long-running")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)
