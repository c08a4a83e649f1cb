import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA library")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def pytest_collection_modifyitems(config, items):
    # GPU tests fail loudly (never skip silently) when selected on a GPU box;
    # on a CPU box they are deselected by the driver's `-m "not gpu"`.
    pass


@pytest.fixture(scope="session")
def tiny_model():
    from synthetic.shapes import get_shape
    from synthetic.weights import make_weights
    from oracle.transformer import Model
    shape = get_shape("tiny")
    w = make_weights(shape, seed=0)
    return shape, w, Model(shape, w.as_f64())
