import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a) and the built libvox.so")
    config.addinivalue_line("markers", "slow: longer CPU test")


def _has_cuda():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _has_cuda():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(autouse=True)
def _debug_bounds_checks(request):
    """With VOX_DEBUG_LIB=1 (the bounds-checked build, tools/debug_checks.sh), every GPU test
    also asserts that no library bounds check fired."""
    yield
    if os.environ.get("VOX_DEBUG_LIB") == "1" and "gpu" in request.keywords:
        import ctypes
        from paper_2604_13191_b200 import lib
        f = ctypes.c_uint32(0)
        assert lib().vox_debug_flags(ctypes.byref(f)) == 0
        assert f.value == 0, f"library bounds checks fired: bits {f.value:#x}"
