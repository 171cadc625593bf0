import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs an sm_100 (B200) GPU and the native library")
    config.addinivalue_line("markers", "slow: full-size (BASELINE config) parity checks")


def pytest_collection_modifyitems(config, items):
    # a kernel that never finishes must fail the test, not hang the GPU box
    for item in items:
        if item.get_closest_marker("gpu") and not item.get_closest_marker("timeout"):
            item.add_marker(pytest.mark.timeout(600))


@pytest.fixture(scope="session", autouse=True)
def _oracle_built():
    # the CPU oracle is test infrastructure; build it on first use
    from oracle import oracle as O
    if not os.path.exists(O.ORACLE_SO):
        O.build()
    # the native library (nvcc cross-compiles sm_100a without a GPU): a fresh
    # checkout gets it built once, incrementally afterwards
    from paper_2604_02570_b200 import build as B
    if not os.path.exists(B.LIB):
        B.build()
    yield
