"""pytest configuration: the ``gpu`` marker and shared fixtures.

``-m "not gpu"`` runs here (no GPU): oracle pins, generator, host logic, C-ABI load/exports,
gloo multi-process sharding.  ``-m gpu`` runs on a B200 and calls the CUDA path through the
C-ABI (``paper_1308_2572_b200``) against the oracle.
"""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) and the built libara.so")
    config.addinivalue_line("markers", "slow: long-running (full-size parity sampling)")


@pytest.fixture(scope="session")
def golden_dir():
    return os.path.join(ROOT, "tests", "golden")
