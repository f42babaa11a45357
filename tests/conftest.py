import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through libctd_gpu.so)")
    config.addinivalue_line("markers", "slow: longer CPU parity runs")


@pytest.fixture(scope="session")
def port():
    from oracle.bindings import Port, build
    build(ref=False)
    return Port()


@pytest.fixture(scope="session")
def ref():
    from oracle.bindings import Ref, ref_available
    if not ref_available():
        pytest.skip("reference oracle not built (oracle/_ref/libctdref.so)")
    return Ref()


@pytest.fixture(scope="session")
def ctx():
    import paper_1710_03608_b200 as ctd
    return ctd.Context(0)
