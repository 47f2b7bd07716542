import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests of the CUDA path")
    config.addinivalue_line("markers", "slow: longer CPU oracle pins")


def _ensure_port():
    from oracle import oracle as O

    if not O.available("port"):
        O.build("port")
    return O


@pytest.fixture(scope="session")
def port():
    O = _ensure_port()
    return O.Oracle("port")


@pytest.fixture(scope="session")
def ref():
    from oracle import oracle as O

    if not O.available("ref"):
        if os.path.isdir("/root/reference/proj/include"):
            O.build("ref")
        else:
            pytest.skip("reference build (oracle/_ref) not available on this box")
    return O.Oracle("ref")


@pytest.fixture(scope="session")
def gpu():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2406_16499_b200 as P

    return P
