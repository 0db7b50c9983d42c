"""Shared fixtures.  `-m gpu` tests call the CUDA path through the C ABI and compare it
with the oracle; everything else runs on CPU (oracle vs golden vectors, host logic,
C-ABI symbol export)."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box)")


@pytest.fixture(scope="session")
def oracle():
    from oracle.bindings import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def ref():
    """The compiled, unmodified reference (oracle/_ref); skipped where it was never built."""
    from oracle.bindings import Ref
    if not Ref.available():
        pytest.skip("reference library not available (no /root/reference and no prebuilt oracle/_ref)")
    return Ref()


@pytest.fixture(scope="session")
def gp():
    import paper_2412_20980_b200 as pkg
    return pkg


@pytest.fixture(scope="session")
def cuda_device(gp):
    import ctypes
    n = ctypes.c_int(0)
    lib = gp.capi.load()
    if lib.gapa_cuda_device_count(ctypes.byref(n)) != 0 or n.value < 1:
        pytest.fail("GPU test selected but no CUDA device is visible — the CUDA path has no fallback")
    return 0
