"""Shared pytest configuration.

Markers: ``gpu`` tests need a B200 (run on the GPU box via gpurun); all other
tests run on the CPU-only build container.
"""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
for p in (ROOT, os.path.join(ROOT, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running test")


GOLDEN_CASES = ("cube10_drop", "cube10_contact", "lat3_contact_drag", "worm",
                "actuated_quiescent", "yield_break", "constraints_contacts",
                "topology_edits", "nan_abort")


def load_golden(name: str) -> dict:
    with np.load(os.path.join(GOLDEN, f"{name}.npz")) as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def golden():
    return load_golden
