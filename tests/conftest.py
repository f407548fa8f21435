import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

BENCH_ARCH = "lstm(5,20,10),softmax(20,3)"
WIDE_ARCH = "lstm(5,20,10),dense(20,4096,relu),dense(4096,4096,relu),softmax(4096,3)"  # SURVEY §8 wide


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as O
    O.lib()
    return O


@pytest.fixture(scope="session")
def ctx():
    import paper_1712_05878_b200 as g
    return g.Context(0)
