import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

REFERENCE_SRC = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs libhmx.so kernels")
    config.addinivalue_line("markers", "slow: long-running")


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


@pytest.fixture(scope="session")
def reference_modules():
    """The reference's own geometry / kernel core, importable only in the
    build container (``/root/reference`` does not exist on the GPU box)."""
    if not os.path.isdir(REFERENCE_SRC):
        pytest.skip("reference mount not present")
    sys.path.insert(0, REFERENCE_SRC)
    try:
        from hmatx import _kernelcore_np, errors, geometry
    finally:
        sys.path.remove(REFERENCE_SRC)
    return geometry, _kernelcore_np, errors
