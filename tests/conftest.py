import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100) device")
    config.addinivalue_line("markers", "slow: long-running case")


@pytest.fixture(scope="session")
def oracle():
    from bindings import COracle
    return COracle()


@pytest.fixture(scope="session")
def ref():
    from bindings import REF_SO, RefOracle
    if not os.path.exists(REF_SO):
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return RefOracle()


@pytest.fixture(scope="session")
def ifgf():
    import paper_2112_15198_b200 as m
    return m


@pytest.fixture(scope="session")
def gpu(ifgf):
    if not ifgf.device_ok():
        raise RuntimeError("gpu test without a usable sm_100 device: " + ifgf._lib.last_error())
    return ifgf
