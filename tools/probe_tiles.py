"""Experiment: per-tile timeline of the select kernel (probe build).
Build: python -c "from paper_2402_13781_b200 import build as B; B.build(defines=['-DEXD_PROBE'], out=B.LIBDIR+'/libexdyna_probe.so')"
Run:   EXD_LIB=paper_2402_13781_b200/lib/libexdyna_probe.so python tools/probe_tiles.py
Phases per tile k: 0 iteration start (loads of k issued), 4 A(k) published,
1/2/3 finish_tile(k) start / prefix known / copy done, 5 extra look-back rounds.
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
S.flush_l2(0, eng.stream())
eng.step([pool[0]])
buf = (C.c_uint64 * (6 * 8192))()
L.exd_debug_tiles(buf)
a = np.frombuffer(buf, dtype=np.uint64).reshape(6, 8192).astype(np.int64)
nt = (n_g + 4095) // 4096
a = a[:, :nt]
rounds = a[5].copy()
t0 = a[0].min()
T = (a[:5] - t0) / 1e3
start, fstart, fprefix, fdone, apub = T
def pct(x):
    return "p50 %.2f p90 %.2f max %.2f" % tuple(np.percentile(x, [50, 90, 100]))
print(f"tiles {nt}; last A {apub.max():.1f} us; last finish {fdone.max():.1f} us")
print("compute (start -> A):", pct(apub - start))
print("A -> finish start:", pct(fstart - apub))
print("look-back (finish start -> prefix):", pct(fprefix - fstart))
print("copy (prefix -> done):", pct(fdone - fprefix))
print("extra rounds: mean %.2f max %d" % (rounds.mean(), rounds.max()))
for i in list(range(0, nt, 150)) + [nt - 1]:
    print(f"tile {i:5d} start {start[i]:6.1f} A {apub[i]:6.1f} fin {fstart[i]:6.1f} pre {fprefix[i]:6.1f} "
          f"done {fdone[i]:6.1f} rounds {rounds[i]}")
