import os
import sys

import pytest

# The one-process emulation of the multi-GPU path (tests/test_dist.py) runs up to 8 ranks'
# persistent kernels concurrently on 8 streams; with the default 8 hardware connections two of
# them can share a queue and serialise (the second never starts while the first waits for it).
# Read by CUDA at context creation, so set before torch initialises CUDA.
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
# ... and a rank's first launch of a kernel instance must not lazily load the module while the
# other ranks' kernels spin (the library also loads each instance before the ranks launch).
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU and the built CUDA library")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)
