import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests through the C ABI")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def port():
    from oracle import Port

    return Port()


@pytest.fixture(scope="session")
def ref():
    from oracle import Ref

    if not Ref.available():
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return Ref()
