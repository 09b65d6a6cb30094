"""Shared pytest setup: the ``gpu`` marker and repo-root imports.

``-m "not gpu"`` runs the oracle-vs-golden checks, host logic, the
multi-process (gloo) sharding tests and the C-ABI export check on CPU;
``-m gpu`` runs the parity tests proper through the CUDA extension.
"""

import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(scope="session")
def golden_small():
    with open(os.path.join(GOLDEN, "golden_small.json")) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def golden_c3():
    path = os.path.join(GOLDEN, "golden_c3.json")
    if not os.path.exists(path):
        pytest.skip("golden_c3.json not generated")
    with open(path) as fh:
        return json.load(fh)
