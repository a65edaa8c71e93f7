import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200) and the built libedkm.so")
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


def pytest_sessionfinish(session, exitstatus):
    """EDKM_PARITY_REPORT=path: the normwise errors every GPU parity check measured, as JSON
    (max and median per quantity, and every sample) -- DESIGN.md S7's measured error distribution."""
    path = os.environ.get("EDKM_PARITY_REPORT")
    mod = sys.modules.get("test_gpu_parity") or sys.modules.get("tests.test_gpu_parity")
    if not path or mod is None or not getattr(mod, "ERRS", None):
        return
    import json
    import statistics
    by = {}
    for test, q, v in mod.ERRS:
        by.setdefault(q, []).append((v, test))
    out = {q: {"n": len(v), "max": max(x for x, _ in v), "median": statistics.median(x for x, _ in v),
               "worst_test": max(v)[1]} for q, v in by.items()}
    with open(path, "w") as f:
        json.dump({"summary": out, "samples": mod.ERRS}, f, indent=1)
