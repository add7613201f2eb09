import os
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


@pytest.fixture(scope="session")
def orc():
    from oracle_py import Oracle  # test infrastructure (the CPU checker)
    return Oracle()


@pytest.fixture(scope="session")
def ref():
    from oracle_py import Reference, OracleError
    try:
        return Reference()
    except OracleError as e:  # /root/reference absent and no prebuilt oracle/_ref
        pytest.skip(str(e))


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")
