"""CPU: the C-ABI library loads, exports every entry point include/exdyna.h
declares, and the ctypes mirror has the header's struct layouts."""
import ctypes as C
import os
import re
import subprocess
import tempfile

import pytest

from paper_2402_13781_b200 import _abi as A
from paper_2402_13781_b200._lib import EXPORTED, LIB_PATH, lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "exdyna.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(exd_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_what_the_binding_uses():
    assert declared_functions() == sorted(EXPORTED)


def test_library_exports_every_declared_symbol():
    out = subprocess.run(["nm", "-D", "--defined-only", LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    syms = {line.split()[-1] for line in out.splitlines() if line.strip()}
    missing = [f for f in declared_functions() if f not in syms]
    assert not missing, missing
    L = lib()
    for f in declared_functions():
        assert hasattr(L, f)


def test_library_has_no_torch_or_oracle_dependency():
    out = subprocess.run(["ldd", LIB_PATH], capture_output=True, text=True).stdout
    assert "torch" not in out and "oracle" not in out and "sparsim_ref" not in out
    out = subprocess.run(["nm", "-D", "--undefined-only", LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "orc_" not in out and "ref_" not in out.replace("pref", "")


def test_version_and_pure_functions_without_gpu():
    L = lib()
    assert L.exd_version() == 1
    assert L.exd_default_block_count(8) == 512


STRUCTS = ["exd_config", "exd_options", "exd_topology", "exd_record", "exd_gather_stats",
           "exd_worker_state", "exd_stream_spec", "exd_kernel_stats"]


def test_struct_layouts_match_header():
    prog = ['#include <stdio.h>', '#include <stddef.h>', '#include "exdyna.h"', "int main(void){"]
    for s in STRUCTS:
        prog.append(f'printf("{s} %zu\\n", sizeof({s}));')
        for fname, _ in getattr(A, s)._fields_:
            prog.append(f'printf("{s}.{fname} %zu\\n", offsetof({s}, {fname}));')
    prog.append("return 0;}")
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "sz.c")
        open(c, "w").write("\n".join(prog))
        exe = os.path.join(d, "sz")
        subprocess.run(["gcc", "-I" + os.path.join(ROOT, "include"), c, "-o", exe], check=True)
        out = subprocess.run([exe], capture_output=True, text=True, check=True).stdout
    got = dict(line.rsplit(" ", 1) for line in out.splitlines())
    for s in STRUCTS:
        cls = getattr(A, s)
        assert int(got[s]) == C.sizeof(cls), s
        for fname, _ in cls._fields_:
            assert int(got[f"{s}.{fname}"]) == getattr(cls, fname).offset, (s, fname)


def test_errors_map_to_reference_exceptions():
    from paper_2402_13781_b200 import sparsim as S
    with pytest.raises(S.InvalidArgument, match="density out of range"):
        S.validate(S.SparsifierConfig(n=2, n_g=64, n_b=2, d=0.0, min_blk=1))
    # engine construction validates before touching the device
    with pytest.raises(S.InvalidArgument, match="^n_b > n_g$"):
        S.Engine(S.SparsifierConfig(n=2, n_g=64, n_b=128, d=0.5, min_blk=1))


def _resources():
    """{mangled kernel name: {REG, STACK, SHARED, LOCAL}} from the sm_100a cubin."""
    exe = "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(exe):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([exe, "--dump-resource-usage", LIB_PATH], capture_output=True,
                         text=True).stdout
    res, name = {}, None
    for line in out.splitlines():
        m = re.search(r"Function (\S+?):?$", line.strip())
        if m:
            name = m.group(1)
            continue
        if name and "REG:" in line:
            res[name] = {k: int(v) for k, v in re.findall(r"(REG|STACK|SHARED|LOCAL):(\d+)", line)}
            name = None
    return res


def test_hot_kernels_compiled_for_sm100a_without_local_memory():
    # the stream kernel (K1) of the headline step (fp32, eta == 1, with and
    # without the NVLink pushes) keeps everything in registers: no stack, no
    # local memory, at most 64 registers (4 CTAs of 256 threads per SM)
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    res = _resources()
    for push in ("0", "1"):
        key = [k for k in res if f"stream_kernelIfLi0ELb1ELb{push}E" in k]
        assert len(key) == 1, key
        r = res[key[0]]
        assert r["STACK"] == 0 and r["LOCAL"] == 0 and r["REG"] <= 64, (key[0], r)
