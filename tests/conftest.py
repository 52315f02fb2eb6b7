import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
TESTS = os.path.dirname(os.path.abspath(__file__))
if TESTS not in sys.path:
    sys.path.insert(0, TESTS)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run on the GPU box via gpurun)")
    config.addinivalue_line("markers", "ref: needs the reference compiled in place (oracle/_ref)")


@pytest.fixture(scope="session")
def ref():
    from oracle import ref as _ref
    if not _ref.available():
        pytest.skip("oracle/_ref not built (reference sources absent)")
    return _ref


@pytest.fixture(scope="session")
def ixo():
    from oracle import ixo as _ixo
    _ixo.lib()
    return _ixo
