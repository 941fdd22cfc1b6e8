import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(Path(__file__).resolve().parent))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200) and the built libalert_b200.so")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def golden_runs():
    from helpers import load_golden_runs
    return load_golden_runs()


@pytest.fixture(scope="session")
def golden_predict():
    from helpers import load_golden_predict
    return load_golden_predict()


@pytest.fixture(scope="session")
def golden_goals():
    from helpers import load_golden_runs
    return load_golden_runs("golden_goals.npz")


@pytest.fixture(scope="session")
def golden_baselines():
    from helpers import load_golden_runs
    return load_golden_runs("golden_baselines.npz")
