import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden" / "reference_conventions.npz"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built libmps_b200.so")


@pytest.fixture(scope="session")
def golden():
    return dict(np.load(GOLDEN))


@pytest.fixture(scope="session")
def c1_sites():
    from oracle import mps_oracle as orc

    return orc.random_mps(8, 16, 4, seed=0)


@pytest.fixture(scope="session")
def c2_sites():
    from oracle import mps_oracle as orc

    return orc.random_mps(16, 100, 10, seed=0)
