"""The C++ facade (include/exdyna/engine.hpp) a sparsim::Engine caller uses:
compiles on CPU (C++17 for the device-buffer API, C++20 for the
GradientSource-driven Engine); on a GPU it replays the reference's
hand-traced row (test_engine.cpp:79-131) through exdyna::Engine, both with
device buffers and with a GradientSource."""
import os
import subprocess

import pytest

from paper_2402_13781_b200._lib import LIB_PATH

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CPP = os.path.join(ROOT, "tests", "cpp")
LIBDIR = os.path.join(ROOT, "paper_2402_13781_b200", "lib")
PROGS = {"engine_facade_golden": "c++17", "engine_source_golden": "c++20"}
CUDA = "/usr/local/cuda"


def _build(name):
    libdir = os.path.dirname(LIB_PATH)
    exe = os.path.join(LIBDIR, name)
    subprocess.run(["g++", "-std=" + PROGS[name], "-O2", "-Wall", "-Werror",
                    "-I" + os.path.join(ROOT, "include"), "-I" + CUDA + "/include",
                    os.path.join(CPP, name + ".cpp"), "-o", exe, "-L" + libdir, "-lexdyna",
                    "-L" + CUDA + "/lib64", "-lcudart", "-Wl,-rpath," + libdir,
                    "-Wl,-rpath," + CUDA + "/lib64"], check=True)
    return exe


@pytest.mark.parametrize("name", sorted(PROGS))
def test_facade_compiles_and_links(name):
    assert os.path.exists(_build(name))


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(PROGS))
def test_facade_on_gpu(name):
    exe = _build(name)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "PASS" in r.stdout
