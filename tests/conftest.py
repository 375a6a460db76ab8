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


def pytest_terminal_summary(terminalreporter, exitstatus, config):
    """Print the session's KLT parity totals (oracle/parity.py SESSION) so a
    test log carries total and attributable status flips."""
    try:
        from oracle import parity
    except Exception:  # pragma: no cover - oracle not importable
        return
    if parity.SESSION["calls"]:
        terminalreporter.write_line(parity.session_summary())
