"""The C++ drop-in facade compiles against the C-ABI (CPU) and reproduces the
reference's results when run on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "facade_demo")


def build():
    lib = os.path.join(ROOT, "paper_1108_1310_b200")
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "facade_demo.cpp"), "-L", lib, "-llamg_b200",
                    f"-Wl,-rpath,{lib}", "-o", BIN], check=True)


def test_facade_compiles_and_links():
    build()
    assert os.path.exists(BIN)


@pytest.mark.gpu
def test_facade_runs_on_gpu(port):
    import numpy as np
    from paper_1108_1310_b200 import graphs as G
    if not os.path.exists(BIN):
        build()
    out = subprocess.run([BIN], check=True, capture_output=True, text=True).stdout.splitlines()
    a = G.grid_5pt(64)
    b = np.zeros(a.n)
    b[0], b[-1] = 1.0, -1.0
    _, st = port.setup(a).solve(b, np.zeros(a.n))
    assert out[0].split()[3] == str(int(st["cycles"][0])), out[0]
    assert out[1].startswith("IncompatibleRhsError: right-hand side sum")
    assert out[2] == "components 3 converged 1 x6 0.0"
    assert out[3] == f"mm n {a.n} m {a.m} same 1 laplacian 0", out[3]
    assert out[4] == "IoError: cannot open: /nonexistent/x.mtx"
