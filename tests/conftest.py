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


@pytest.fixture
def set_options(sg):
    """set_options(kernel="mixed", ...) for the rest of the test (sg_set_options);
    the previous process-wide options are restored at teardown."""
    import ctypes as C
    from paper_2208_09985_b200 import _ffi
    L = _ffi.load()
    saved = _ffi.SgOptions()
    L.sg_get_options(C.byref(saved))

    def setter(**kw):
        cm = sg.options(**kw)
        cm.__enter__()  # restored below, not by the context manager

    yield setter
    L.sg_set_options(C.byref(saved))
