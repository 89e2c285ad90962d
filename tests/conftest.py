"""Shared test setup.

Markers: `gpu` = needs a CUDA device (B200); everything else runs on CPU.
The oracle (oracle/mtb_oracle.py) and the golden vectors (tests/golden/) are
the checkers; the product package never imports them.
"""

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: requires a CUDA device (sm_100a); run with -m gpu")


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(GOLDEN_DIR, "golden.json")) as f:
        meta = json.load(f)
    arrays = dict(np.load(os.path.join(GOLDEN_DIR, "golden.npz")))
    return meta, arrays


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("GPU test selected but no CUDA device is visible")
    return torch


@pytest.fixture(autouse=True)
def _reset_counters():
    try:
        from paper_2007_06483_b200.instrumentation import counters
    except Exception:  # pragma: no cover
        yield
        return
    counters.reset()
    yield
