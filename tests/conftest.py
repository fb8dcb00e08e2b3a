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
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a); run with -m gpu")


@pytest.fixture(scope="session")
def orc():
    from _oracle import oracle

    return oracle()


@pytest.fixture(scope="session")
def ref():
    from _oracle import reference

    r = reference()
    if r is None:
        pytest.skip("oracle/_ref (reference built from /root/reference) not present")
    return r
