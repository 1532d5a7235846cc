import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = Path(__file__).resolve().parent / "golden"
sys.path.insert(0, str(ROOT))

BOUNDS = {
    "f1": (-5.12, 5.12), "f2": (-5.12, 5.12), "f3": (-65.536, 65.536), "f4": (-2.048, 2.048),
    "f5": (-5.12, 5.12), "f6": (-32.768, 32.768), "f7": (-600.0, 600.0), "f8": (-4.0, 5.0),
    "f9": (-5.12, 5.12),
}
# objectives whose device/oracle fitness is bitwise by construction (pure +,-,*
# in numpy order); the others use transcendentals whose libm results differ by ulps
BITWISE_FIDS = ("f1", "f2", "f3", "f4")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def golden_runs():
    index = json.loads((GOLDEN / "runs.json").read_text())
    arrays = np.load(GOLDEN / "runs.npz")
    return index, arrays


@pytest.fixture(scope="session")
def golden_fitness():
    return np.load(GOLDEN / "fitness.npz")


@pytest.fixture(scope="session")
def golden_rng():
    return np.load(GOLDEN / "rng.npz")


@pytest.fixture(scope="session")
def golden_seq_runs():
    """Reference run_sequential results (tests/golden/make_seq_golden.py)."""
    index = json.loads((GOLDEN / "seq_runs.json").read_text())
    arrays = np.load(GOLDEN / "seq_runs.npz")
    return index, arrays
