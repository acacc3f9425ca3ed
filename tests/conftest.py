"""Shared test configuration.

* registers the ``gpu`` marker (tests that need a B200; run with ``-m gpu``);
* the deterministic hypothesis profile of the reference suite
  (reference pkg/tests/conftest.py:5-12);
* puts the repo root on sys.path so ``oracle`` and the package import.
"""

import os
import sys

import pytest
from hypothesis import HealthCheck, settings

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

settings.register_profile(
    "ci",
    derandomize=True,
    max_examples=200,
    deadline=None,
    suppress_health_check=[HealthCheck.too_slow],
)
settings.load_profile("ci")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200) and the built library")


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda", 0)
