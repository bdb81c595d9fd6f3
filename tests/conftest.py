import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def port():
    """The plain-C restatement (oracle/atk_oracle.c), built on demand."""
    from oracle import pyoracle as O
    if not os.path.exists(O.PORT_PATH):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "port"], check=True, capture_output=True)
    return O.port()


@pytest.fixture(scope="session")
def ref():
    """The reference library compiled from /root/reference (oracle/_ref)."""
    from oracle import pyoracle as O
    if not O.ref_available() and os.path.isdir("/root/reference/proj/core"):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "ref"], check=True, capture_output=True)
    if not O.ref_available():
        pytest.skip("oracle/_ref/libatk_ref.so not available")
    return O.ref()


@pytest.fixture(scope="session")
def stage_fixtures():
    return np.load(os.path.join(ROOT, "tests", "golden", "stage_fixtures.npz"))


@pytest.fixture(scope="session")
def planner_fixtures():
    return np.load(os.path.join(ROOT, "tests", "golden", "planner_fixtures.npz"), allow_pickle=True)


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")
