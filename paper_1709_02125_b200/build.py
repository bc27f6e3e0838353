"""Build the two native libraries of ooc-b200 in-tree (paper_1709_02125_b200/lib/).

  liboocdev.so  CUDA device layer (include/ooc_device.h) — nvcc, sm_100a only
  libooc.so     C++ host engine: planner, lazy runtime, streaming executor, apps and
                the runtime C ABI (include/ooc_stencil.h); links liboocdev.so

Field parity with the reference is bit-exact, so floating-point contraction is
disabled on both sides (nvcc --fmad=false, g++ -ffp-contract=off, no -march).
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "lib")
OBJ = os.path.join(LIB, "obj")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
CXX = "/usr/bin/g++"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
INC = ["-I" + os.path.join(ROOT, "include"), "-I" + os.path.join(CSRC, "include")]

DEV_SRCS = ["device/ooc_device.cu", "device/loop_kernels.cu", "device/jit.cu", "device/sweep.cu",
            "device/comm.cu"]
HOST_SRCS = ["host/core.cpp", "host/tiler.cpp", "host/runtime.cpp", "host/gpu_engine.cpp",
             "host/apps.cpp", "host/capi.cpp", "host/metrics.cpp", "host/chain_file.cpp", "host/seams.cpp"]
HEADERS_DEV = ["device/internal.cuh", "device/jit.cuh"]
HEADERS_HOST = ["host/json_writer.hpp", "host/json_reader.hpp"] + [os.path.join("include/ooc", h)
                                            for h in os.listdir(os.path.join(CSRC, "include/ooc"))]

NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "--fmad=false", "-std=c++17", "-Xcompiler", "-fPIC",
                     "-Xptxas", "-warn-spills"] + INC
CXX_FLAGS = ["-std=c++20", "-O2", "-fPIC", "-fopenmp", "-ffp-contract=off", "-Wall", "-Wextra",
             "-Wno-unused-parameter"] + INC + ["-I/usr/local/cuda/include"]


def _newest(paths):
    return max(os.path.getmtime(p) for p in paths if os.path.exists(p))


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("build failed:\n" + " ".join(cmd) + "\n" + r.stdout + r.stderr)
    return r.stdout + r.stderr


def _compile(src, dev):
    s = os.path.join(CSRC, src)
    o = os.path.join(OBJ, os.path.basename(src) + ".o")
    deps = [s] + [os.path.join(CSRC, h) for h in (HEADERS_DEV if dev else HEADERS_HOST)] + \
        [os.path.join(ROOT, "include", h) for h in os.listdir(os.path.join(ROOT, "include"))]
    if os.path.exists(o) and os.path.getmtime(o) >= _newest(deps):
        return o, ""
    cmd = ([NVCC] + NVCC_FLAGS if dev else [CXX] + CXX_FLAGS) + ["-c", s, "-o", o]
    return o, _run(cmd)


def build(verbose=False, jobs=8):
    os.makedirs(OBJ, exist_ok=True)
    with cf.ThreadPoolExecutor(jobs) as ex:
        dev = list(ex.map(lambda s: _compile(s, True), DEV_SRCS))
        host = list(ex.map(lambda s: _compile(s, False), HOST_SRCS))
    for _, log in dev + host:
        if verbose and log:
            print(log)
    devlib = os.path.join(LIB, "liboocdev.so")
    dobjs = [o for o, _ in dev]
    if not os.path.exists(devlib) or os.path.getmtime(devlib) < _newest(dobjs):
        _run([NVCC] + ARCH + ["-shared", "-o", devlib] + dobjs + ["-cudart", "static", "-ldl"])
    hostlib = os.path.join(LIB, "libooc.so")
    hobjs = [o for o, _ in host]
    if not os.path.exists(hostlib) or os.path.getmtime(hostlib) < _newest(hobjs + [devlib]):
        _run([CXX, "-shared", "-fopenmp", "-Wl,-Bsymbolic", "-o", hostlib] + hobjs +
             ["-L" + LIB, "-loocdev", "-Wl,-rpath,$ORIGIN"])
    return devlib, hostlib


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
