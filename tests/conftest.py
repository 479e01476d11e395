import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running GPU case")


@pytest.fixture(scope="session")
def golden():
    import numpy as np

    cache = {}

    def load(name):
        if name not in cache:
            path = os.path.join(GOLDEN, name)
            if name.endswith(".json"):
                import json
                with open(path) as fh:
                    cache[name] = json.load(fh)
            else:
                cache[name] = dict(np.load(path, allow_pickle=False))
        return cache[name]

    return load


@pytest.fixture
def triangle():
    from paper_2604_26423_b200 import WmcInstance
    return WmcInstance(3, ((0, 1, 0.5), (0, 2, 1.0), (1, 2, 0.25)))
