import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def lc():
    from oracle.oracle import LC_LIB, LcOracle, build_oracles

    if not LC_LIB.exists():
        build_oracles(with_ref=False)
    return LcOracle()


@pytest.fixture(scope="session")
def ref():
    from oracle.oracle import RefOracle, ref_available

    if not ref_available():
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return RefOracle()


def golden(name):
    return dict(np.load(GOLDEN / f"{name}.npz"))
