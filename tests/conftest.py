import sys
from pathlib import Path

import numpy as np
import pytest

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
GOLDEN = REPO / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu on the GPU box)")


@pytest.fixture(scope="session")
def golden():
    return dict(np.load(GOLDEN / "golden.npz"))


@pytest.fixture(scope="session")
def payloads():
    return dict(np.load(GOLDEN / "golden_payloads.npz"))


@pytest.fixture(scope="session")
def cfg0_stream():
    return (GOLDEN / "streams" / "cfg0.hivc").read_bytes()


@pytest.fixture(scope="session")
def cfg0_frames():
    return np.load(GOLDEN / "cfg0_frames.npz")["frames"]


@pytest.fixture(scope="session")
def enc_golden():
    return dict(np.load(GOLDEN / "golden_encoder.npz"))
