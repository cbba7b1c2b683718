"""bench.py — ExDyna sparsify+sync on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (N > 1)

One step = one Engine::step() (engine.cpp:274-350) of the ExDyna sparsifier
over one ResNet-18-sized fp32 gradient per worker (configs[1] of BASELINE.json:
n_g = 11.2M, d = 0.01, n_b = 256), one worker per GPU. Gradients are synthetic
(the reference's default four-segment Laplace stream, seed 7, generated on the
device) and already resident in HBM for `value`; `e2e` runs the same steps
through the public C ABI from pinned host buffers with the H2D copies inside
the timed region. L2 is flushed before every timed step (a 2x-L2 buffer is
written, then read back so no dirty lines land on the next kernel).

--impl reference times the UNMODIFIED reference (oracle/_ref, compiled from
/root/reference/proj/src) on the host cores: rank 0 simulates all N workers in
one process with the reference's own worker threads, as sparsim does.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_G = 11_200_000
DENSITY = 0.01
N_B = 256
SEED = 7
METRIC = "sparsify+sync ms/iter (ExDyna step, R18 n_g=11.2M, d=0.01)"
UNIT = "ms/iter"
POOL = 2  # gradient buffers per worker: step t reads one while t+1's is generated


def cfg_kw(n):
    # every parameter pinned (SURVEY.md §7 hard part 10)
    return dict(n=n, n_g=N_G, n_b=N_B, d=DENSITY, alpha=1.25, beta=1.25, gamma=0.02,
                blk_move=1, min_blk=2, eta=1.0, seed=SEED)


def workload(n):
    return {"workload": "configs[1]: ResNet-18-sized gradient, partitioned sparsify+sync",
            "n_g": N_G, "d": DENSITY, "k": round(DENSITY * N_G), "n_b": N_B, "workers": n,
            "alpha": 1.25, "beta": 1.25, "gamma": 0.02, "min_blk": 2, "blk_move": 1,
            "delta0": "auto (t=0 quantile)", "stream": "default 4-segment Laplace, seed 7",
            "l2": "flushed before every timed step (2x L2 buffer written, then read back)", "parallelism": f"dp{n}",
            "sync": "single GPU" if n == 1 else None}


# ------------------------------------------------------------------ clocks --
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        sm = [float(r[1]) for r in self.rows if len(r) > 8 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) > 8 and r[2].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            if len(r) > 8:
                for nm, v in zip(names, r[5:9]):
                    if v.lower().startswith("active"):
                        reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic():
    """dram bytes per fused-select launch from the committed ncu --set full summary."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "ncu_select_*.json")))
    if not files:
        return None
    try:
        d = json.load(open(files[-1]))
        return d.get("dram_bytes_per_launch")
    except Exception:
        return None


def max_over_ranks(values, dist=None):
    """Max of each timing over all ranks (the contract's whole-job time): the
    slowest rank defines the step. `dist` is torch.distributed or None."""
    if dist is None:
        return [float(v) for v in values]
    import torch
    t = torch.tensor([float(v) for v in values], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(v) for v in t]


# ------------------------------------------------------- reference (CPU) ----
def host_cpu():
    """CPU model and core count of this host (for the baseline's context)."""
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return f"{model}, nproc={os.cpu_count()}"


def reference_ms_per_step(n, steps, warmup, pool=None):
    """Time the unmodified reference's Engine::step() (oracle/_ref) on this host."""
    import numpy as np
    from oracle import oracle as O
    if not O.ref_available():
        raise RuntimeError("oracle/_ref/libsparsim_ref.so not built")
    cfg = O.make_config(**cfg_kw(n))
    pool = pool or n
    eng = O.RefEngine(cfg, O.make_options(), pool=pool)  # as shipped: threads + verify_replication
    spec = O.stream_spec(N_G, None, seed=SEED)
    for s in range(pool):
        g = O.synthetic_gradient_orc(spec, s // n, s % n).astype(np.float32)
        eng.set_slot(s, g)
    for _ in range(warmup):
        eng.step()
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        eng.step()
        times.append((time.perf_counter() - t0) * 1e3)
    return statistics.mean(times), times


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    n = args.gpus
    steps = max(1, min(args.steps, 30))
    warmup = max(1, min(args.warmup, 3))
    try:
        ms, _ = reference_ms_per_step(n, steps, warmup)
    except Exception as e:  # the reference is always buildable here; report why not
        print(json.dumps({"impl": "reference", "unavailable": str(e)}))
        return 0
    cores = n  # sparsim runs n-1 worker threads + the caller (engine.cpp:90-117)
    line = {
        "metric": METRIC, "value": ms, "unit": UNIT, "n_gpus": n, "steps": steps, "warmup": warmup,
        "ms_per_step": ms, "higher_is_better": False, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic", "impl": "reference", "config": workload(n),
        "cpu_baseline": {"value": ms, "unit": UNIT, "cores": cores, "kind": "reference",
                         "sample": f"full R18 Engine::step() with {n} simulated workers, "
                                   f"{steps} timed steps after {warmup} warm-up "
                                   f"(verify_replication on, worker threads on; {host_cpu()})"},
        "e2e": {"value": ms, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


# ------------------------------------------------------------------ ours ----
def run_ours(args):
    import numpy as np
    import torch

    from paper_2402_13781_b200 import sparsim as S

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    n = args.gpus
    if world != n:
        raise SystemExit(f"--gpus {n} but WORLD_SIZE={world}; launch N>1 with torchrun")
    torch.cuda.set_device(local)
    dist = None
    if n > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")  # control plane only; the data path is NCCL in C++
    kw = cfg_kw(n)
    opt = S.EngineOptions(dtype="f32", profile_kernels=False, verify_replication=False,
                          record_loss=False, sync=args.sync)
    if n == 1:
        eng = S.Engine(S.SparsifierConfig(**kw), opt, device=local)
    else:
        obj = [S.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        eng = S.Engine.rank(S.SparsifierConfig(**kw), opt, rank, local, obj[0])
    stream = torch.cuda.ExternalStream(eng.stream())
    src = S.SyntheticStream(S.StreamSpec(n_g=N_G, seed=SEED))
    bufs = [torch.empty(N_G, dtype=torch.float32, device=f"cuda:{local}") for _ in range(POOL)]
    for i, b in enumerate(bufs):
        src.gradient(i, rank, b, "f32", eng.stream())
    torch.cuda.synchronize()

    def barrier():
        torch.cuda.synchronize()
        if dist:
            dist.barrier()

    clocks = ClockSampler(local)
    clocks.start()
    # warm-up: W steps, then enough more for ~1.5 s under load so the clock
    # samples see it; every rank must run the same number of steps (each step
    # is a set of collectives), so rank 0 decides and broadcasts the count
    i = 0

    def run_steps(k):
        nonlocal i
        for _ in range(k):
            src.gradient(i, rank, bufs[i % POOL], "f32", eng.stream())  # fresh g_t (untimed)
            eng.step_async([bufs[i % POOL]])
            if i % 16 == 15:
                eng.sync()
            i += 1
        eng.sync()

    t0 = time.time()
    run_steps(args.warmup)
    per_step = max((time.time() - t0) / args.warmup, 1e-5)
    extra = [int(min(1.5 / per_step, 200_000))]
    if dist:
        t = torch.tensor(extra)
        dist.broadcast(t, src=0)
        extra = [int(t[0])]
    run_steps(extra[0])
    # ---- value: K steps, each bracketed by events on the engine's stream, L2
    # flushed before each (flush excluded). Per-kernel profiling is OFF here so
    # the stream->finish programmatic launch overlap is what gets timed.
    eng.set_profile(False)
    eng.reset_kernel_stats()
    S.flush_l2(local, eng.stream())  # first call allocates the flush buffer (a device sync)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    for a_, b_ in ev:  # torch creates CUDA events lazily, at the first record
        a_.record(stream)
        b_.record(stream)
    run_steps(1)
    per_step_launches = eng.kernel_stats()["kernel_launches"]
    launches0 = per_step_launches + 2 * per_step_launches  # the two aligning steps below
    barrier()
    # two untimed steps enqueued right behind the host barrier, with no host
    # sync before the timed ones: the ranks leave the barrier up to ~0.2 ms
    # apart, and the steps' in-kernel exchange realigns their streams
    for _ in range(2):
        src.gradient(i, rank, bufs[i % POOL], "f32", eng.stream())
        eng.step_async([bufs[i % POOL]])
        i += 1

    recs = []
    for k in range(args.steps):
        src.gradient(i + k, rank, bufs[(i + k) % POOL], "f32", eng.stream())  # untimed
        S.flush_l2(local, eng.stream())
        ev[k][0].record(stream)
        eng.step_async([bufs[(i + k) % POOL]])
        ev[k][1].record(stream)
        if k % 8 == 7:
            recs.append(eng.sync())
    recs.append(eng.sync())
    barrier()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    if os.environ.get("EXD_BENCH_VERBOSE"):
        srt = sorted(step_ms)
        print(f"[rank {rank}] step ms: mean {statistics.mean(step_ms):.4f} min {srt[0]:.4f} "
              f"median {srt[len(srt) // 2]:.4f} max {srt[-1]:.4f} first5 "
              f"{[round(v, 4) for v in step_ms[:5]]}", file=sys.stderr, flush=True)
    ks = eng.kernel_stats()
    launches = ks["kernel_launches"] - launches0
    total_ms = sum(step_ms)
    i += args.steps

    # ---- roofline: the same steps with CUDA events around each kernel ----
    eng.set_profile(True)
    eng.reset_kernel_stats()
    prof_steps = max(10, min(args.steps, 50))
    for k in range(prof_steps):
        src.gradient(i + k, rank, bufs[(i + k) % POOL], "f32", eng.stream())
        S.flush_l2(local, eng.stream())
        eng.step_async([bufs[(i + k) % POOL]])
        if n > 1 or k % 8 == 7:
            recs.append(eng.sync())
    i += prof_steps
    ks2 = eng.kernel_stats()
    sel_ms = ks2["select_ms"] / max(ks2["select_launches"], 1)
    fin_ms = ks2["finish_ms"] / max(ks2["finish_launches"], 1)
    eng.set_profile(False)
    total_ms, sel_ms, fin_ms = max_over_ranks([total_ms, sel_ms, fin_ms], dist)
    ms = total_ms / args.steps

    # ---- e2e: public API from pinned host buffers, H2D inside the region ----
    host = []
    for b in bufs[:2]:
        h = torch.empty(N_G, dtype=torch.float32, pin_memory=True)
        h.copy_(b.cpu())
        host.append(h)
    import ctypes as C
    from paper_2402_13781_b200 import _abi as A
    from paper_2402_13781_b200._lib import check, lib
    L = lib()
    rec = A.exd_record()
    e2e_steps = max(3, min(args.steps, 20))
    ev2 = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(e2e_steps)]
    for a_, b_ in ev2:
        a_.record(stream)
        b_.record(stream)
    # one untimed call first: it allocates the engine's device staging buffer
    check(L.exd_engine_step_host(eng.h, (C.c_void_p * 1)(host[1].data_ptr()), C.byref(rec)))
    barrier()
    for k in range(e2e_steps):
        S.flush_l2(local, eng.stream())
        ev2[k][0].record(stream)
        ptrs = (C.c_void_p * 1)(host[k % 2].data_ptr())
        check(L.exd_engine_step_host(eng.h, ptrs, C.byref(rec)))  # returns with the record on the host
        ev2[k][1].record(stream)
    barrier()
    if os.environ.get("EXD_BENCH_VERBOSE"):
        print(f"[rank {rank}] e2e ms: {[round(a.elapsed_time(b), 3) for a, b in ev2]}",
              file=sys.stderr, flush=True)
    e2e_total = max_over_ranks([sum(a.elapsed_time(b) for a, b in ev2)], dist)[0]
    e2e_ms = e2e_total / e2e_steps
    clk = clocks.stop()

    if rank != 0:
        if dist:
            dist.barrier()
        return 0

    # roofline of the dominant kernel (fused accumulate+select+compact)
    kp = statistics.mean(r.k_prime for r in recs)
    k_own = statistics.mean(r.k_rank[0] for r in recs)
    alg_bytes = 12 * N_G + 8 * k_own + (8 * kp if n == 1 else 0)
    achieved = alg_bytes / (sel_ms * 1e-3) / 1e9
    peak, peak_src = peaks()
    traffic = ncu_traffic()
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": traffic, "kernel": "stream_kernel<float,kFused> (K1: accumulate + select + stage)",
            "kernel_ms": sel_ms, "finish_kernel_ms": fin_ms,
            "algorithmic_bytes_per_launch": alg_bytes,
            "peak_source": peak_src, "share_of_step": sel_ms / ms}

    cpu = None
    if n == 1:
        try:
            cms, _ = reference_ms_per_step(1, 5, 1, pool=2)
            cpu = {"value": cms, "unit": UNIT, "cores": 1, "kind": "reference",
                   "sample": "5 full R18 n=1 Engine::step() calls of the unmodified reference "
                             "(oracle/_ref) after 1 warm-up, replayed fp32-rounded gradients; "
                             + host_cpu()}
        except Exception as e:
            cpu = {"value": None, "unit": UNIT, "cores": 1, "kind": "reference",
                   "sample": f"unavailable: {e}"}

    # sync stage over NVLink (push-reduce): algorithmic bytes each GPU stores into
    # its peers' inboxes per step, against the exchange kernel's event time
    nvlink = None
    if n > 1 and eng.sync_mode() == "p2p":
        tiles_own = (N_G / n) / 4096.0
        holder = (n >= 4) if "EXD_HOLDER_SUM" not in os.environ else os.environ["EXD_HOLDER_SUM"] == "1"
        words = (kp - k_own) + (n - 1) * k_own if holder else (n - 1) * kp  # contribution/sum words out
        out_b = (n - 1) * (8 * k_own + 72 * tiles_own) + 8 * words
        nvlink = {"bytes_out_per_gpu_per_step": out_b, "sync_kernel_ms": fin_ms,
                  "achieved_gbs": out_b / (fin_ms * 1e-3) / 1e9, "peak_gbs": 900.0,
                  "frac": out_b / (fin_ms * 1e-3) / 1e9 / 900.0,
                  "note": "latency-bound at this size (~1 MB per GPU per step): the exchange "
                          "kernel's time is round trips, not link bandwidth; bytes = staged-index "
                          "and count words pushed by the stream kernel + 8 B contribution words "
                          "(to every peer, or to the holder and sums back for n >= 4)",
                  "holder_sum": holder}
    cfg_line = workload(n)
    if n > 1:
        cfg_line["sync"] = {
            "p2p": "NVLink peer memory, push-reduce (lists pushed during the stream, "
                   "everything as {payload, epoch} words; no handshake, no host wait)",
            "p2p-pull": "NVLink peer memory, pull-reduce (lists pushed, contributions pulled)",
            "nccl": "NCCL all-gather/all-reduce + one host wait"}[eng.sync_mode()]
    line = {
        "metric": METRIC, "value": ms, "unit": UNIT, "n_gpus": n, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic", "config": cfg_line,
        "selection_hbm_gbs": achieved,
        "roofline": roof,
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_ms, "unit": UNIT, "h2d_bytes_per_step": 4 * N_G * n,
                "d2h_bytes_per_step": C.sizeof(A.exd_record) * n},
        "gpu_launches": launches,
        "nvlink": nvlink,
        "clocks": clk,
        "records": {"k_prime_mean": kp, "f_t_mean": statistics.mean(r.f_t for r in recs),
                    "density_mean": statistics.mean(r.density for r in recs),
                    "t_last": recs[-1].t},
        "step_ms_min": min(step_ms), "step_ms_median": statistics.median(step_ms),
        "step_ms_p90": sorted(step_ms)[int(0.9 * (len(step_ms) - 1))], "step_ms_max": max(step_ms),
    }
    print(json.dumps(line))
    if dist:
        dist.barrier()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--sync", default="auto", choices=["auto", "nccl", "p2p", "p2p-pull"],
                    help="N > 1: NVLink peer-memory sync (auto/p2p) or the NCCL chain")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
