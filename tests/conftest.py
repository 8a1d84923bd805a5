"""Shared pytest setup: the ``gpu`` marker and import paths.

``-m "not gpu"`` runs on the CPU build container (oracle vs golden vectors,
host logic, C-ABI symbol table, gloo multi-process bookkeeping);
``-m gpu`` runs the parity tests proper on a B200.
"""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
for p in (ROOT, os.path.join(ROOT, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


def cuda_ok():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture
def golden_dir():
    return GOLDEN
