import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (runs on the B200 box)")


@pytest.fixture(scope="session")
def orc():
    from oracle.oracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def ref():
    from oracle.oracle import Reference, have_reference
    if not have_reference():
        pytest.skip("oracle/_ref/libsvdbref.so not built (reference sources absent)")
    return Reference()


@pytest.fixture(scope="session")
def gpu():
    import paper_2504_04564_b200 as P
    if P.device_count() < 1:
        pytest.fail("no CUDA device visible: gpu tests must run on the B200 box")
    return P
