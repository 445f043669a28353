"""Shared test configuration: the ``gpu`` marker and fixtures.

Tests marked ``gpu`` need a B200 and the built CUDA library; everything else
runs on CPU (the oracle, host-side logic, the C-ABI symbol table, gloo
multi-process tests).
"""

from __future__ import annotations

import os
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
for p in (ROOT, HERE):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200) and the built libnnm.so")


@pytest.fixture
def rng():
    return np.random.default_rng(0xC0FFEE)
