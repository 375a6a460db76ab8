"""Shared pytest configuration.

Markers: ``gpu`` — needs a CUDA device (run on the B200 box via gpurun);
everything else must pass on a CPU-only machine.
"""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


@pytest.fixture(scope="session")
def cuda_available():
    import torch
    return torch.cuda.is_available()
