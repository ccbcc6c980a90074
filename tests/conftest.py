import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running parity sweep")
    # Build the product library and the oracle once if this checkout lacks them
    # (nvcc cross-compiles without a GPU; gcc builds the oracle).
    # (build.py is loaded by path: the package itself refuses to import
    # without its .so)
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "_lmdtw_build", os.path.join(ROOT, "paper_2008_02734_b200", "build.py"))
    _b = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(_b)
    if not os.path.exists(_b.LIB):
        _b.build()
    from oracle import oracle as _o
    _o.build()


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
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)
