"""Shared pytest config. `-m "not gpu"` runs on the CPU dev box; `-m gpu`
runs on a B200 (via gpurun) and FAILS (never skips) when no GPU is visible,
so a silent CPU run cannot pass for a GPU run."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU; run via gpurun")
    config.addinivalue_line("markers", "slow: long-running (full-size oracle) test")


@pytest.fixture(autouse=True)
def _require_gpu_for_gpu_tests(request):
    if request.node.get_closest_marker("gpu") is not None:
        import torch
        if not torch.cuda.is_available():
            pytest.fail("gpu-marked test needs a visible CUDA device (run under gpurun)")
    yield
