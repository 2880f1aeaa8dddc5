import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs the sm_100a engine")


@pytest.fixture(scope="session")
def engine():
    from paper_2411_14968_b200 import Engine
    e = Engine(0)
    yield e
    e.close()


@pytest.fixture(scope="session")
def golden():
    import json
    import numpy as np
    here = os.path.join(ROOT, "tests", "golden")
    with open(os.path.join(here, "golden.json")) as f:
        g = json.load(f)
    g["plane_arrays"] = np.load(os.path.join(here, "plane.npz"))
    g["plane64_arrays"] = np.load(os.path.join(here, "plane64.npz"))
    g["config_arrays"] = np.load(os.path.join(here, "configs.npz"))
    return g


@pytest.fixture
def options(engine):
    """Set engine options (sky_ctx_set_option) for one test; defaults after."""
    def set_(**kw):
        for k, v in kw.items():
            engine.set_option(k, v)
    yield set_
    engine.reset_options()
