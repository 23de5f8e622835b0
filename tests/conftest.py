import os
import sys

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
for p in (HERE, ROOT):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100) device; run with -m gpu")
    config.addinivalue_line("markers", "slow: longer CPU oracle checks")


@pytest.fixture(scope="session")
def kat():
    import json
    with open(os.path.join(HERE, "golden", "kat.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def engine():
    """One device context for the GPU tests (fails loudly without a device)."""
    import paper_2006_16783_b200 as T
    e = T.Engine(0)
    yield e
    e.close()


@pytest.fixture(scope="session")
def c1_terrain():
    """BASELINE config 1's terrain (1000x1000, roughness 0.5, 0..4000), oracle-generated."""
    import oracle_lib as O
    return O.generate_fractal(1000, 1000, 0.5, 1, 0, 4000)
