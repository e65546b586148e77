import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the sm_100a kernels)")
    config.addinivalue_line("markers", "slow: long-running (full-size) case")


def pytest_sessionstart(session):
    # build the native libraries if they are missing (no-op when up to date)
    from paper_1309_1889_b200 import build as b
    lib = ROOT / "paper_1309_1889_b200" / "lib"
    if not (lib / "libmsmb.so").exists() or not (lib / "libmsmb_fixtures.so").exists() \
            or not (ROOT / "oracle" / "liboracle.so").exists():
        b.build_all()


@pytest.fixture(scope="session")
def port():
    import oracle_lib
    return oracle_lib.checker("port")


@pytest.fixture(scope="session")
def ref():
    import oracle_lib
    if not oracle_lib.have("ref"):
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return oracle_lib.checker("ref")


def golden(name):
    return dict(np.load(GOLDEN / f"{name}.npz", allow_pickle=False))


def rel_rms(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.sqrt(np.sum((a - b) ** 2) / max(np.sum(b ** 2), 1e-300)))


def rel_e(a, b):
    return abs(a - b) / abs(b)
