"""A C++ loop chain written against the reference API compiles unchanged against the
ooc-b200 headers and runs on the GPU with results identical to the oracle."""
import os
import subprocess

import numpy as np
import pytest

from oracle import ooc_oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_1709_02125_b200")


def build_example(tmp_path):
    exe = str(tmp_path / "heat_chain")
    subprocess.run(["/usr/bin/g++", "-std=c++20", "-O2", "-ffp-contract=off",
                    "-I", os.path.join(PKG, "csrc", "include"), "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "examples", "heat_chain.cpp"), "-o", exe,
                    "-L", os.path.join(PKG, "lib"), "-looc", "-Wl,-rpath," + os.path.join(PKG, "lib")],
                   check=True)
    return exe


def test_example_compiles(tmp_path):
    assert os.path.exists(build_example(tmp_path))


@pytest.mark.gpu
def test_example_runs_on_gpu_bitwise(tmp_path):
    exe = build_example(tmp_path)
    n, iters = 96, 7
    r = subprocess.run([exe, str(n), str(iters), "3"], capture_output=True, check=True)
    got = np.frombuffer(r.stdout, dtype=np.float64)
    rt = O.Runtime("reference")
    u = rt.declare("u", O.Ext.make(2, (0, 0), (n, n)), (1, 1), 8, "(+ 1.0 (* 0.125 (+ i j)))")
    t = rt.declare("tmp", O.Ext.make(2, (0, 0), (n, n)), (1, 1), 8, 0.0)
    s5 = [(0, 0, 0), (-1, 0, 0), (1, 0, 0), (0, -1, 0), (0, 1, 0)]
    avg = O.parse_prefix("(* 0.25 (+ (+ (r 0 -1 0) (r 0 1 0)) (+ (r 0 0 -1) (r 0 0 1))))")
    for _ in range(iters):
        rt.enqueue_loop(O.Loop(O.Ext.make(2, (1, 1), (n - 1, n - 1)),
                               [O.Arg(u, s5, O.READ), O.Arg(t, [(0, 0, 0)], O.WRITE)], [(1, avg)]))
        rt.enqueue_loop(O.Loop(O.Ext.make(2, (1, 1), (n - 1, n - 1)),
                               [O.Arg(t, [(0, 0, 0)], O.READ), O.Arg(u, [(0, 0, 0)], O.WRITE)],
                               [(1, ("read", 0, (0, 0, 0)))]))
    want = rt.fetch_dataset(u).ravel()
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))
    usum = float(r.stderr.decode().split()[1])
    assert abs(usum - want[(want.size and 0):].reshape(n + 2, n + 2)[1:-1, 1:-1].sum()) <= 1e-9 * usum
