import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

try:  # same hypothesis profile as the reference suite (tests/conftest.py:5-11 there)
    from hypothesis import HealthCheck, settings

    settings.register_profile("suite", max_examples=50, deadline=None,
                              suppress_health_check=[HealthCheck.too_slow])
    settings.load_profile("suite")
except ImportError:  # pragma: no cover
    pass


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture
def rng():
    # seeded Philox stream, as the reference fixture (tests/conftest.py:14-16 there)
    return np.random.Generator(np.random.Philox(20260824))


@pytest.fixture(scope="session")
def golden():
    path = os.path.join(ROOT, "tests", "golden", "golden.npz")
    with np.load(path) as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def golden_meta():
    import json

    with open(os.path.join(ROOT, "tests", "golden", "golden_meta.json")) as fh:
        return json.load(fh)
