import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through the CUDA C ABI)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def orc():
    from oracle.bindings import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def ref():
    """The reference library itself; only where oracle/_ref was built."""
    from oracle.bindings import REF_SO, Ref
    if not os.path.exists(REF_SO):
        pytest.skip("oracle/_ref/libspecmoe_ref.so not built")
    return Ref()
