"""pytest configuration: the `gpu` marker and shared fixtures.

`-m "not gpu"` runs on the CPU-only container (oracle vs golden vectors, host
logic, ABI exports); `-m gpu` runs on a B200 and exercises the CUDA library
through its C ABI against the CPU oracle.
"""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests through the C ABI")
    config.addinivalue_line("markers", "slow: larger parity cases")


def _has_gpu():
    try:
        import ctypes
        rt = ctypes.CDLL("libcuda.so.1")
        n = ctypes.c_int(0)
        if rt.cuInit(0) != 0:
            return False
        return rt.cuDeviceGetCount(ctypes.byref(n)) == 0 and n.value > 0
    except OSError:
        return False


HAS_GPU = _has_gpu()


@pytest.fixture(scope="session")
def gpu_ctx():
    if not HAS_GPU:
        pytest.fail("test marked gpu but no CUDA device is visible")
    from paper_2605_26137_b200 import capi
    return capi.default_context()


@pytest.fixture(scope="session")
def port():
    from oracle import bindings
    return bindings.port()


@pytest.fixture(scope="session")
def ref():
    from oracle import bindings
    if not bindings.ref_available():
        pytest.skip("oracle/_ref not built (reference sources absent)")
    return bindings.ref()
