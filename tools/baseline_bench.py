"""Time the device baseline sparsifiers at the R18 size.

    python tools/baseline_bench.py [--n 11200000] [--k 112000] [--iters 50]

Each call is timed with CUDA events on the current stream around the whole C
ABI call (scratch alloc, radix select, count, scan, emit, count read-back).
Algorithmic bytes per call: hard threshold 2 reads of acc + 4 B per index;
top-k adds one read of acc per 11-bit radix pass (3 for f32, 6 for f64).
Peak: MEASURED_PEAKS.json hbm_gbs.
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2402_13781_b200 import sparsim as S  # noqa: E402


def timed(fn, iters, flush):
    ts = []
    for _ in range(iters):
        flush.fill_(1.0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=11_200_000)
    ap.add_argument("--k", type=int, default=112_000)
    ap.add_argument("--iters", type=int, default=50)
    args = ap.parse_args()
    peak = 6650.0  # B200_PROFILING.md fallback when MEASURED_PEAKS.json is absent
    try:
        peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(
            os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"]
    except Exception:
        pass
    flush = torch.empty(64 << 20, device="cuda:0")  # 256 MB > L2
    for dt, esz, passes in ((torch.float32, 4, 3), (torch.float64, 8, 6)):
        acc = torch.distributions.Laplace(0.0, 1.0).sample((args.n,)).to("cuda:0", dt)
        delta = float(acc.abs().float().kthvalue(args.n - args.k + 1).values)
        for _ in range(3):
            S.topk_select(acc, args.k)
            S.hard_threshold_select(acc, delta)
        torch.cuda.synchronize()
        for name, fn, nbytes in (
                ("topk_select", lambda: S.topk_select(acc, args.k),
                 (2 + passes) * esz * args.n + 4 * args.k),
                ("hard_threshold_select", lambda: S.hard_threshold_select(acc, delta),
                 2 * esz * args.n + 4 * args.k)):
            ms = timed(fn, args.iters, flush)
            gbs = nbytes / ms / 1e6
            print(json.dumps({"op": name, "dtype": str(dt).split(".")[-1], "n_g": args.n,
                              "k": args.k, "ms": ms, "algorithmic_bytes": nbytes,
                              "achieved_gbs": gbs, "peak_gbs": peak, "frac": gbs / peak}))


if __name__ == "__main__":
    main()
