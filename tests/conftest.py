import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running full-size parity case")


@pytest.fixture
def rng():
    return np.random.default_rng(1234)


@pytest.fixture
def square_target():
    from paper_2006_10509_b200.workloads import square_target as make

    return make
