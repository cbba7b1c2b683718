"""Experiment: per-CTA timeline of the finish kernel's copy CTAs (probe build).
Build: python -c "from paper_2402_13781_b200 import build as B; B.build(defines=['-DEXD_PROBE'], out=B.LIBDIR+'/libexdyna_probe.so')"
Run:   EXD_LIB=paper_2402_13781_b200/lib/libexdyna_probe.so python tools/probe_ctas.py
"""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2402_13781_b200 import sparsim as S
from paper_2402_13781_b200._lib import lib
L = lib()
n_g = 11_200_000
eng = S.Engine(S.SparsifierConfig(n=1, n_g=n_g, n_b=256, d=0.01, seed=7), S.EngineOptions())
src = S.SyntheticStream(S.StreamSpec(n_g=n_g, seed=7))
pool = [torch.empty(n_g, device="cuda") for _ in range(2)]
for i, b in enumerate(pool):
    src.gradient(i, 0, b, "f32", eng.stream())
for i in range(200):
    eng.step_async([pool[i % 2]])
eng.sync()
for rep in range(4):
    S.flush_l2(0, eng.stream())
    eng.step([pool[rep % 2]])
    pb = (C.c_uint64 * 64)()
    L.exd_debug_probe(pb)
    buf = (C.c_uint64 * (4 * 2048))()
    L.exd_debug_ctas(buf)
    a = np.frombuffer(buf, dtype=np.uint64).reshape(4, 2048).astype(np.int64)
    G = int((a[0] > 0).sum())
    a = a[:, :G]
    t0 = pb[16]
    start, based, done = [(x - t0) / 1e3 for x in a[:3]]
    ent = a[3]
    k1end = (pb[31] - t0) / 1e3
    def pct(x):
        return "p50 %.1f p90 %.1f max %.1f" % tuple(np.percentile(x, [50, 90, 100]))
    print(f"rep {rep}: G={G} K1_END {k1end:.1f}  entries {pct(ent)} total {ent.sum()}")
    print(f"  start {pct(start)}  base {pct(based)}  done {pct(done)}  copy {pct(done - based)}")
    slow = np.argsort(done)[-5:]
    print("  slowest:", [(int(i), round(float(done[i]), 1), int(ent[i])) for i in slow])
    print("  corr(entries, copy time) = %.2f" % np.corrcoef(ent, done - based)[0, 1])
