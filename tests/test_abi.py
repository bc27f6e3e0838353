"""The C-ABI libraries load on CPU and export every symbol include/*.h declares."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_1709_02125_b200", "lib")


def declared(header):
    text = open(os.path.join(ROOT, "include", header)).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ooc_[a-z0-9_]+)\s*\(", text)))


@pytest.mark.parametrize("header,lib", [("ooc_device.h", "liboocdev.so"),
                                        ("ooc_stencil.h", "libooc.so")])
def test_exports(header, lib):
    L = ctypes.CDLL(os.path.join(LIBDIR, lib))
    names = declared(header)
    assert len(names) > 10
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing


def test_device_layer_reports_no_device_cleanly():
    L = ctypes.CDLL(os.path.join(LIBDIR, "liboocdev.so"))
    n = ctypes.c_int(-1)
    rc = L.ooc_dev_count(ctypes.byref(n))
    assert rc in (0, -12)
    L.ooc_dev_build_info.restype = ctypes.c_char_p
    assert b"sm_100a" in L.ooc_dev_build_info()


def test_sass_is_sm100a():
    """The device library carries sm_100a SASS (cuobjdump), no other arch."""
    import shutil
    import subprocess
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(tool):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([tool, "--list-elf", os.path.join(LIBDIR, "liboocdev.so")],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out
