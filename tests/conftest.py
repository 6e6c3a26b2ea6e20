"""Shared pytest configuration.

Markers: ``gpu`` = needs a B200 (run with ``-m gpu``); everything else runs
on CPU in a few minutes (``-m "not gpu"``).
"""
from __future__ import annotations

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: requires a CUDA B200 device (sm_100a)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def golden_lines(name: str):
    """Non-comment, non-empty lines of a golden fixture."""
    with open(os.path.join(GOLDEN, name)) as f:
        return [ln.strip() for ln in f if ln.strip() and not ln.lstrip().startswith("#")]


def golden_matrix(name: str) -> np.ndarray:
    return np.array([[float(t) for t in ln.split()] for ln in golden_lines(name)])


@pytest.fixture(scope="session")
def orc():
    import oracle
    oracle.build()
    return oracle
