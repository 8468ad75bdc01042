from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest

REPO = Path(__file__).resolve().parent.parent
GOLDEN = REPO / "tests" / "golden"
sys.path.insert(0, str(REPO))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs an sm_100 GPU (runs on the B200 box)")
    config.addinivalue_line("markers", "slow: long-running")


def unravel(sizes, flat):
    out, o = [], 0
    for n in sizes:
        n = int(n)
        out.append(flat[o:o + n * n].reshape(n, n).copy())
        o += n * n
    return out


def load_golden(name: str) -> dict:
    with np.load(GOLDEN / name) as z:
        return {k: z[k] for k in z.files}


def has_gpu() -> bool:
    try:
        from paper_1707_02423_b200 import _native
        return _native.device_count() > 0
    except Exception:
        return False


@pytest.fixture(scope="session")
def gpu():
    if not has_gpu():
        pytest.fail("no sm_100 GPU visible: GPU tests must run on the B200 box")
    return 0
