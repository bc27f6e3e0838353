"""Test configuration: `gpu` marks tests that need a B200 (run with -m gpu)."""
import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(scope="session")
def golden_random():
    with open(os.path.join(GOLDEN, "random_programs.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def golden_apps():
    with open(os.path.join(GOLDEN, "apps.json")) as f:
        return json.load(f)


def has_gpu():
    try:
        import ctypes
        n = ctypes.c_int()
        lib = ctypes.CDLL("libcudart.so.12")
        return lib.cudaGetDeviceCount(ctypes.byref(n)) == 0 and n.value > 0
    except OSError:
        return False
