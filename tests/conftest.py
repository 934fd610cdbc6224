import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu on the GPU box)")


@pytest.fixture(scope="session")
def cuda():
    """The native library on a real device; fails loudly (no skip, no fallback)."""
    from paper_2212_08146_b200 import native

    n = native.device_count()
    assert n > 0, "no CUDA device visible: GPU tests must run on the B200 box"
    native.init_device(0)
    return native
