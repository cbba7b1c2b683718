"""Experiment: phase timestamps (globaltimer) of the stream/finish kernels.
Build: python -c "from paper_2402_13781_b200 import build as B; B.build(defines=['-DEXD_PROBE'], out=B.LIBDIR+'/libexdyna_probe.so')"
Run:   EXD_LIB=paper_2402_13781_b200/lib/libexdyna_probe.so python tools/probe_finish.py [--n 1]
"""
import argparse, ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
ap = argparse.ArgumentParser(); ap.add_argument("--n", type=int, default=1); a = ap.parse_args()
import torch
from paper_2402_13781_b200 import sparsim as S
from paper_2402_13781_b200._lib import lib
L = lib()
L.exd_debug_probe.argtypes = [C.POINTER(C.c_uint64)]
n_g = 11_200_000
eng = S.Engine(S.SparsifierConfig(n=a.n, n_g=n_g, n_b=256, d=0.01, seed=7),
               S.EngineOptions(verify_replication=False))
src = S.SyntheticStream(S.StreamSpec(n_g=n_g, seed=7))
pool = [[torch.empty(n_g, device="cuda") for _ in range(a.n)] for _ in range(2)]
for i, bs in enumerate(pool):
    for r, b in enumerate(bs):
        src.gradient(i, r, b, "f32", eng.stream())
torch.cuda.synchronize()
for i in range(300):
    eng.step_async(pool[i % 2])
eng.sync()
names = {4: "epi_warm", 0: "epi_start", 1: "epi_sums", 2: "epi_pre_cta",
         3: "epi_end", 8: "copy0_start", 9: "copy0_base", 10: "copyL_base", 11: "copy0_end",
         12: "copyL_end", 16: "k1_first_cta", 17: "k1_last_cta", 26: "epi_delta", 27: "epi_plan",
         28: "epi_record", 30: "K2_END", 31: "K1_END"}
rows = []
xs = torch.cuda.ExternalStream(eng.stream())
for i in range(5):
    S.flush_l2(0, eng.stream())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(xs)
    eng.step_async(pool[i % 2])
    e1.record(xs)
    eng.sync()
    buf = (C.c_uint64 * 64)()
    L.exd_debug_probe(buf)
    zero = (C.c_uint64 * 64)()
    t0 = buf[16]
    row = {names[k]: (buf[k] - t0) / 1e3 for k in names if buf[k]}
    row["EVENTS_us"] = e0.elapsed_time(e1) * 1e3
    rows.append(row)
for r in rows:
    print("  ".join(f"{k}={v:.1f}" for k, v in sorted(r.items(), key=lambda kv: kv[1])))
# back to back (no flush, no sync between steps): the gap from the finish
# kernel's last stamp of step t to the stream kernel's first CTA of step t+1
xs2 = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(50)]
for i in range(50):
    xs2[i][0].record(xs)
    eng.step_async(pool[i % 2])
    xs2[i][1].record(xs)
eng.sync()
buf = (C.c_uint64 * 64)()
L.exd_debug_probe(buf)
us = sorted(a_.elapsed_time(b_) * 1e3 for a_, b_ in xs2)
print(f"back-to-back: step median {us[25]:.1f} us; prev step k1 -> K2_END {(buf[52] - buf[51]) / 1e3:.1f} us, "
      f"K2_END -> this k1 {(buf[16] - buf[52]) / 1e3:.1f} us")
