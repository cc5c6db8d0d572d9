import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests")):
    if p not in sys.path:
        sys.path.insert(0, p)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (CUDA device) and the built det library")
    config.addinivalue_line("markers", "live_reference: needs /root/reference importable (build container only)")


def cuda_available() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    from refshim import reference_available

    skip_ref = pytest.mark.skip(reason="reference package not present")
    has_ref = reference_available()
    for it in items:
        if "live_reference" in it.keywords and not has_ref:
            it.add_marker(skip_ref)


@pytest.fixture(scope="session")
def golden_dir():
    return GOLDEN


@pytest.fixture(autouse=True)
def _device_guard_zones(request):
    """Under DET_GUARD=1 (the library's guard-zone debug mode) every GPU test ends with a check that
    no device buffer's guard zone was overwritten (compute-sanitizer is not available on the pool)."""
    yield
    if os.environ.get("DET_GUARD", "0") == "0" or "gpu" not in request.keywords:
        return
    import ctypes

    from paper_2604_13880_b200 import _lib

    live, bad = ctypes.c_longlong(0), ctypes.c_longlong(0)
    rc = _lib.load_library().det_debug_guard_check(ctypes.byref(live), ctypes.byref(bad))
    assert rc == 0, "DET_GUARD set but the library's guard mode is off"
    assert bad.value == 0, f"{bad.value} device guard zone(s) overwritten ({live.value} live buffers)"
