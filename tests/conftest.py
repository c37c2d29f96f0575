"""Shared test plumbing.

``-m "not gpu"`` runs here (no GPU): the oracle against the reference's golden
fixtures, the host-side API, the C-ABI library's exported symbols, and the
gloo multi-process sharding logic.  ``-m gpu`` runs on a B200 and compares the
CUDA path (through ``libctqw.so``) with the oracle.
"""

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libctqw.so")


def load_golden(name):
    data = np.load(os.path.join(GOLDEN, name))
    meta = json.loads(str(data["meta"]))
    return data, meta


@pytest.fixture(scope="session")
def cuda_device():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("gpu-marked test needs a CUDA device")
    return torch.device("cuda:0")
