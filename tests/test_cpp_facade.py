"""The C++ facade (include/exdyna/engine.hpp) a sparsim::Engine caller uses:
compiles on CPU; on a GPU it replays the reference's hand-traced row
(test_engine.cpp:79-131) through exdyna::Engine."""
import os
import subprocess

import pytest

from paper_2402_13781_b200._lib import LIB_PATH

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "engine_facade_golden.cpp")
EXE = os.path.join(ROOT, "paper_2402_13781_b200", "lib", "engine_facade_golden")
CUDA = "/usr/local/cuda"


def _build():
    libdir = os.path.dirname(LIB_PATH)
    subprocess.run(["g++", "-std=c++17", "-O1", "-I" + os.path.join(ROOT, "include"),
                    "-I" + CUDA + "/include", SRC, "-o", EXE, "-L" + libdir, "-lexdyna",
                    "-L" + CUDA + "/lib64", "-lcudart", "-Wl,-rpath," + libdir,
                    "-Wl,-rpath," + CUDA + "/lib64"], check=True)


def test_facade_compiles_and_links():
    _build()
    assert os.path.exists(EXE)


@pytest.mark.gpu
def test_facade_hand_traced_row_on_gpu():
    if not os.path.exists(EXE):
        _build()
    r = subprocess.run([EXE], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "PASS" in r.stdout
