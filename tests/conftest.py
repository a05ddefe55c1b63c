import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        have_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        have_gpu = False
    if have_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(autouse=True)
def _device_checks(request):
    """With HP_CHECKED=1 (and HP_LIB pointing at libhp_b200_checked.so, the
    `make checked` build): every GPU test must leave no failed device-side
    bounds / invariant check behind."""
    yield
    if os.environ.get("HP_CHECKED") != "1" or "gpu" not in request.keywords:
        return
    import torch

    from paper_2404_14044_b200 import _lib
    torch.cuda.synchronize()
    lines = _lib.check_failures(reset=True)
    assert not lines, f"device-side checks failed at source lines {lines}"
