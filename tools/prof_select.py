"""Profiling driver: R18 (n_g=11.2M, d=0.01) steps on cuda:0 for ncu / timing.

    python tools/prof_select.py [--n N] [--steps S] [--warmup W] [--dtype f32]

Prints per-kernel CUDA-event timing of the fused select kernel (engine
profile_kernels) so a plain run and the ncu capture use the same command.
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1)
    ap.add_argument("--n_g", type=int, default=11_200_000)
    ap.add_argument("--d", type=float, default=0.01)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=400)
    ap.add_argument("--dtype", default="f32")
    ap.add_argument("--flush", type=int, default=1)
    a = ap.parse_args()
    import torch
    from paper_2402_13781_b200 import sparsim as S
    cfg = S.SparsifierConfig(n=a.n, n_g=a.n_g, n_b=256, d=a.d, seed=7)
    eng = S.Engine(cfg, S.EngineOptions(dtype=a.dtype, profile_kernels=True, verify_replication=False))
    td = torch.float64 if a.dtype == "f64" else torch.float32
    src = S.SyntheticStream(S.StreamSpec(n_g=a.n_g, seed=7))
    pool = [[torch.empty(a.n_g, dtype=td, device="cuda") for _ in range(a.n)] for _ in range(2)]
    for i, bs in enumerate(pool):
        for r, b in enumerate(bs):
            src.gradient(i, r, b, a.dtype, eng.stream())
    torch.cuda.synchronize()
    for i in range(a.warmup):
        eng.step(pool[i % 2])
    eng.reset_kernel_stats()
    for i in range(a.steps):
        if a.flush:
            S.flush_l2(0, eng.stream())
        eng.step_async(pool[i % 2])
    rec = eng.sync()
    st = eng.kernel_stats()
    # whole-step time with profiling off (stream->finish launches overlap)
    eng.set_profile(False)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(a.steps)]
    xs = torch.cuda.ExternalStream(eng.stream())
    for i in range(a.steps):
        if a.flush:
            S.flush_l2(0, eng.stream())
        evs[i][0].record(xs)
        eng.step_async(pool[i % 2])
        evs[i][1].record(xs)
    eng.sync()
    step_us = sorted(e0.elapsed_time(e1) * 1e3 for e0, e1 in evs)
    ms = st["select_ms"] / max(1, st["select_launches"])
    byt = (12 if a.dtype == "f32" else 24) * a.n_g
    fin = st["finish_ms"] / max(1, st["finish_launches"])
    print(f"n={a.n} n_g={a.n_g} {a.dtype} stream avg {ms*1e3:.1f} us over {st['select_launches']} launches "
          f"-> {byt/ms/1e6:.0f} GB/s ({byt/a.n_g:.0f} B/elem); finish avg {fin*1e3:.1f} us; "
          f"k'={rec.k_prime} f_t={rec.f_t:.3f} t={rec.t}; step median {step_us[len(step_us)//2]:.1f} us "
          f"(min {step_us[0]:.1f})")


if __name__ == "__main__":
    main()
