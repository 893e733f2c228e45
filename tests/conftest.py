"""Shared fixtures.  GPU tests carry @pytest.mark.gpu; the CPU suite runs
with -m "not gpu".  The C oracle (oracle/) is the parity checker; it is
built on demand."""

import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = ROOT / "tests" / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the CUDA library")


@pytest.fixture(scope="session")
def kernels_golden():
    return np.load(GOLDEN / "kernels.npz")


@pytest.fixture(scope="session")
def solves_golden():
    return json.loads((GOLDEN / "solves.json").read_text()), np.load(GOLDEN / "solves.npz")


@pytest.fixture(scope="session")
def dist_golden():
    return json.loads((GOLDEN / "dist.json").read_text()), np.load(GOLDEN / "dist.npz")


@pytest.fixture(scope="session")
def strategies_golden():
    return json.loads((GOLDEN / "strategies.json").read_text())


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as O

    O.lib()
    return O
