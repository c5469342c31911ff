"""Shared pytest setup.

``-m gpu`` tests need a B200 and the built CUDA library; everything else runs
on the CPU-only build container.  The oracle (oracle/, test infrastructure) is
imported here only as the checker.
"""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libttb.so")
    config.addinivalue_line("markers", "slow: long-running case")


@pytest.fixture(scope="session")
def coracle():
    from oracle import COracle
    return COracle()


@pytest.fixture(scope="session")
def refo():
    from oracle import RefOracle, have_ref
    if not have_ref():
        pytest.skip("reference build oracle/_ref absent")
    return RefOracle()
