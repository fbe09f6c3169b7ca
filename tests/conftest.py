import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the sm_100a CUDA path)")
    config.addinivalue_line("markers", "slow: longer parity runs")


@pytest.fixture(scope="session")
def port():
    from oracle.bindings import CpuChecker
    return CpuChecker("port")


@pytest.fixture(scope="session")
def ref():
    from oracle.bindings import CpuChecker, reference_available
    if not reference_available():
        pytest.skip("oracle/_ref/libdho2ref.so not built (needs /root/reference at build time)")
    return CpuChecker("reference")


@pytest.fixture(scope="session")
def ctx():
    import paper_2505_00982_b200 as d
    c = d.Context(0)
    yield c
    c.close()
