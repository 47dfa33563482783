import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) device")
    config.addinivalue_line("markers", "slow: long CPU test")


@pytest.fixture(scope="session")
def oracle():
    from oracle import pyoracle

    if not os.path.exists(pyoracle.ORACLE_SO):
        pyoracle.build(ref=False)
    return pyoracle.Oracle()


@pytest.fixture(scope="session")
def reflib():
    from oracle import pyoracle

    if not os.path.exists(pyoracle.REF_SO):
        if os.path.isdir("/root/reference"):
            pyoracle.build(ref=True)
        else:
            pytest.skip("oracle/_ref not built and /root/reference absent")
    return pyoracle.RefLib()
