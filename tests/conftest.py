import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box)")


def _cuda_device_count() -> int:
    import ctypes

    for name in ("libcudart.so", "libcudart.so.12"):
        try:
            rt = ctypes.CDLL(name)
        except OSError:
            continue
        n = ctypes.c_int(0)
        if rt.cudaGetDeviceCount(ctypes.byref(n)) == 0:
            return n.value
        return 0
    return 0


@pytest.fixture(scope="session")
def gpu_available():
    return _cuda_device_count() > 0


@pytest.fixture(scope="session")
def oracle():
    from checkers import Oracle

    return Oracle()


@pytest.fixture(scope="session")
def ref():
    from checkers import Ref, have_ref

    if not have_ref():
        pytest.skip("oracle/_ref/libhfmm_ref.so not built (needs /root/reference)")
    return Ref()


@pytest.fixture(scope="session", autouse=True)
def _built_library():
    from paper_1803_09948_b200 import build_library

    build_library()


def pytest_terminal_summary(terminalreporter):
    # a CUDA error some other user of the process left behind (the library clears it at entry)
    try:
        import ctypes

        from paper_1803_09948_b200.api import load_library
        lib = load_library()
        lib.hfmm_debug_stale_cuda_error.restype = ctypes.c_char_p
        stale = lib.hfmm_debug_stale_cuda_error()
        if stale and _cuda_device_count() > 0:
            terminalreporter.write_line("hfmm: stale CUDA error seen at API entry: " + stale.decode())
    except Exception:
        pass
