import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device; runs the sm_100a path")


@pytest.fixture(scope="session")
def sg():
    import paper_2208_09985_b200 as mod
    from paper_2208_09985_b200 import _ffi
    _ffi.load()
    return mod


@pytest.fixture(scope="session")
def gpu(sg):
    from paper_2208_09985_b200 import _ffi
    if _ffi.load().sg_device_count() < 1:
        pytest.fail("no CUDA device visible: GPU tests must run on the B200 box")
    return sg
