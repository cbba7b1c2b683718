"""Build libexdyna.so (the B200 ExDyna path) in-tree with nvcc for sm_100a.

    python -m paper_2402_13781_b200.build

The library has no torch dependency: plain CUDA runtime (static) + NCCL
loaded with dlopen on first multi-GPU use.
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "lib")
LIB = os.path.join(LIBDIR, "libexdyna.so")
SOURCES = ["kernels.cu", "baselines.cu", "baseline_engine.cu", "engine.cu", "ledger.cpp"]
HEADERS = ["control.cuh", "internal.cuh"]

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ARCH + [
    "-O3", "-lineinfo", "-std=c++17", "-Xptxas", "-v",
    "-Xcompiler", "-fPIC,-ffp-contract=off,-O3",
    "-I" + os.path.join(ROOT, "include"), "-I" + CSRC,
]


def _stale():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, s) for s in SOURCES + HEADERS]
    deps.append(os.path.join(ROOT, "include", "exdyna.h"))
    deps.append(os.path.abspath(__file__))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force=False, verbose=False, defines=(), out=None):
    """Compile and link. `defines`/`out` build an experiment variant (e.g.
    -DEXD_PROBE into lib/libexdyna_probe.so) without touching the product."""
    lib_out = out or LIB
    if not force and not defines and not _stale():
        return LIB
    os.makedirs(LIBDIR, exist_ok=True)
    objs = []
    tag = "" if not defines else "_" + "_".join(d.lstrip("-D").lower() for d in defines)
    for src in SOURCES:
        obj = os.path.join(LIBDIR, os.path.splitext(src)[0] + tag + ".o")
        cmd = [NVCC] + FLAGS + list(defines) + ["-c", os.path.join(CSRC, src), "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("nvcc failed on " + src)
        if verbose:
            sys.stderr.write(r.stderr)
        with open(obj + ".ptxas.txt", "w") as f:
            f.write(r.stderr)
        objs.append(obj)
    tmp = lib_out + ".tmp"
    cmd = [NVCC] + ARCH + ["-shared", "-o", tmp] + objs + ["-ldl"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc link failed")
    os.replace(tmp, lib_out)
    return lib_out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
