import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
HERE = os.path.dirname(os.path.abspath(__file__))
if HERE not in sys.path:
    sys.path.insert(0, HERE)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs an sm_100 GPU (run on the B200 box)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def olib():
    from oracle_bind import load_oracle
    return load_oracle()


@pytest.fixture(scope="session")
def ref():
    from oracle_bind import load_ref
    r = load_ref()
    if r is None:
        pytest.skip("oracle/_ref/libcarma_ref.so not built (needs /root/reference)")
    return r


@pytest.fixture(scope="session")
def gpu():
    from paper_2508_19073_b200 import abi
    if abi.lib.carma_device_count() < 1:
        pytest.fail("no sm_100 device: GPU tests must run on the B200 box")
    return 0
