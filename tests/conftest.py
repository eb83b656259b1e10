import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))  # tests may use the oracle as the checker

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


def _ensure_built():
    lib = os.path.join(ROOT, "paper_2304_08662_b200", "_lib", "libxdrop_b200.so")
    ora = os.path.join(ROOT, "oracle", "liboracle.so")
    if not (os.path.exists(lib) and os.path.exists(ora)):
        import subprocess
        subprocess.check_call(["make", "-s", "-C", ROOT, "lib", "oracle"])


_ensure_built()


@pytest.fixture(scope="session")
def oracle():
    from oracle_py import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def golden_dir():
    return GOLDEN


@pytest.fixture(scope="session")
def has_gpu():
    from paper_2304_08662_b200 import capi
    return capi.lib().xb_device_count() > 0


@pytest.fixture(autouse=True)
def _bounds_checks(request):
    """With XB_LIB_PATH pointing at the checked library (make checked), every
    GPU test also asserts that no device-side bounds check failed."""
    yield
    if "gpu" not in request.keywords or "checked" not in os.environ.get("XB_LIB_PATH", ""):
        return
    import ctypes
    from paper_2304_08662_b200 import capi
    failed = ctypes.c_uint32(0)
    rc = capi.lib().xb_debug_checks(0, ctypes.byref(failed))
    assert rc == 0, "XB_LIB_PATH names a library without checks"
    assert failed.value == 0, f"device bounds check {failed.value} failed (xb_kernels.cuh kChk* ids)"
