import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def _cuda_device_count() -> int:
    """Driver-API probe (no torch import: keeps the CPU suite torch-free)."""
    import ctypes
    try:
        cuda = ctypes.CDLL("libcuda.so.1")
    except OSError:
        return 0
    if cuda.cuInit(0) != 0:
        return 0
    n = ctypes.c_int(0)
    if cuda.cuDeviceGetCount(ctypes.byref(n)) != 0:
        return 0
    return n.value


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through libckmpm_b200.so)")
    config.addinivalue_line("markers", "slow: long-running")


def pytest_collection_modifyitems(config, items):
    have_gpu = _cuda_device_count() > 0
    if have_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)
