"""Shared pytest setup.

Markers: ``gpu`` — needs a B200 (run with ``-m gpu`` through gpurun); every
other test runs on the CPU build container.
"""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 device")


def seeded_prompt(seed, length, vocab):
    """tests/conftest.py:24-27 of the reference."""
    rng = np.random.default_rng(seed)
    return [int(x) for x in rng.integers(0, vocab, size=length)]


@pytest.fixture(scope="session")
def golden():
    import json
    arrs = np.load(os.path.join(GOLDEN_DIR, "shiftsim_golden.npz"))
    with open(os.path.join(GOLDEN_DIR, "shiftsim_golden.json")) as f:
        meta = json.load(f)
    return arrs, meta


def c1_prompts():
    """C1 workload: default_rng(7), 8 lengths in [32, 129)."""
    rng = np.random.default_rng(7)
    lens = [int(x) for x in rng.integers(32, 129, size=8)]
    return [[int(t) for t in rng.integers(0, 256, size=n)] for n in lens]
