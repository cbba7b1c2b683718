"""tools/sweep.py — the configs[4] scaling sweep (BASELINE.json): one bench.py
line per cell, n_g in {1M, 10M, 100M, 1B} x d in {0.001, 0.01, 0.1}, at N GPUs.

    python tools/sweep.py --gpus 1 --out profiles/sweep_r02.jsonl
    python tools/sweep.py --gpus 2 --cells 100M:0.01,1B:0.1 ...

Each cell runs `bench.py --n_g X --density d` in its own process (torchrun for
N > 1), so every line carries the same fields as the headline bench line:
device-timed ms/iter (max over ranks), K1's event-timed roofline and, at N = 1,
ncu DRAM bytes of K1 measured in the run (--traffic-cells) and the CPU
reference on the same gradients (--cpu-cells). Lines go to --out as they
finish (one JSON object per line, with the cell's wall time).
"""
import argparse
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SIZES = {"1M": 1_000_000, "10M": 10_000_000, "100M": 100_000_000, "1B": 1_000_000_000}
DENS = [0.001, 0.01, 0.1]


def parse_cells(s):
    if not s:
        return [(k, d) for k in SIZES for d in DENS]
    out = []
    for c in s.split(","):
        k, d = c.split(":")
        out.append((k, float(d)))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--cells", default="")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "sweep_r02.jsonl"))
    ap.add_argument("--cpu-cells", default="1M,10M,100M",
                    help="sizes whose CPU reference is timed (N = 1 only)")
    ap.add_argument("--traffic-cells", default="100M,1B", help="sizes with in-run ncu traffic")
    ap.add_argument("--sync", default="auto")
    ap.add_argument("--port", type=int, default=29531)
    args = ap.parse_args()
    cpu_cells = set(args.cpu_cells.split(",")) if args.cpu_cells else set()
    tr_cells = set(args.traffic_cells.split(",")) if args.traffic_cells else set()
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    for size, d in parse_cells(args.cells):
        n_g = SIZES[size]
        steps = 100 if n_g <= 10_000_000 else 50 if n_g <= 100_000_000 else 20
        bench = [os.path.join(ROOT, "bench.py"), "--gpus", str(args.gpus), "--steps", str(steps),
                 "--warmup", "5", "--n_g", str(n_g), "--density", str(d), "--no-variants",
                 "--sync", args.sync, "--cpu-budget", "10",
                 "--cpu", "auto" if (args.gpus == 1 and size in cpu_cells) else "none",
                 "--traffic", "ncu" if (args.gpus == 1 and size in tr_cells) else "none"]
        if args.gpus == 1:
            cmd = [sys.executable] + bench
        else:
            cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                   f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
                   "--master-port", str(args.port)] + bench
            args.port += 1
        t0 = time.time()
        r = subprocess.run(cmd, capture_output=True, text=True, cwd=ROOT)
        wall = time.time() - t0
        line = None
        for ln in r.stdout.splitlines():
            if ln.startswith("{"):
                line = json.loads(ln)
        if line is None:
            line = {"cell": f"{size}:{d}", "n_gpus": args.gpus, "error": f"rc={r.returncode}",
                    "stderr": r.stderr[-1500:]}
        line["cell"] = f"{size}:{d}"
        line["cell_wall_s"] = round(wall, 1)
        with open(args.out, "a") as f:
            f.write(json.dumps(line) + "\n")
        v = line.get("value")
        roof = line.get("roofline") or {}
        print(f"{size:>5} d={d:<6} N={args.gpus}: "
              + (f"{v * 1e3:9.1f} us/iter  K1 {roof.get('frac', 0):.3f} of HBM  "
                 f"traffic={roof.get('traffic')}" if v else line.get("error", "?"))
              + f"  ({wall:.0f} s)", flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
