"""bench.py — ExDyna sparsify+sync on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (N > 1)
    python bench.py --n_g 100000000 --density 0.1 ...      (a configs[4] sweep cell)

One step = one Engine::step() (engine.cpp:274-350) of the ExDyna sparsifier
over one synthetic gradient per worker, one worker per GPU. The default is
configs[1] of BASELINE.json: the ResNet-18-sized gradient (n_g = 11.2M),
d = 0.01, n_b = 256, fp32. `--n_g/--density/--dtype/--beta/--stream` select
the other configs (GN skew, the configs[4] sweep cells, fp64, beta = 1.05).
Gradients are the reference's Laplace stream generated on the device and
already resident in HBM for `value`; `e2e` runs the same steps through the
public C ABI from pinned host buffers with the H2D copies inside the timed
region. L2 is flushed before every timed step (a 2x-L2 buffer is written,
then read back so no dirty lines land on the next kernel).

At N = 1 the line also carries:
  cpu_baseline  the unmodified reference (oracle/_ref, compiled from
                /root/reference/proj/src) timed on this host, BASELINE.md §3:
                median over up to 50 steps after 5 warm-up steps, "as shipped"
                (verify_replication on, worker threads on) and "lean"
                (verify off, record_loss off), plus the fp32 C restatement
                (the bit-exact checker of the fp32 GPU path);
  roofline      K1's event-timed algorithmic GB/s against MEASURED_PEAKS.json,
                and `traffic` = DRAM bytes of K1 measured by ncu IN THIS RUN
                (a child process under `ncu --metrics dram__bytes_*`);
  variants      (default config only) the fp64 GPU path and beta = 1.05, each
                with its density next to the reference's own on the same
                inputs.

--impl reference times the UNMODIFIED reference (oracle/_ref) on the host
cores: rank 0 simulates all N workers in one process with the reference's
own worker threads, as sparsim does.
"""
import argparse
import json
import os
import shutil
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

R18_N_G = 11_200_000
N_B = 256
SEED = 7
UNIT = "ms/iter"
POOL = 2  # gradient buffers per worker: step t reads one while t+1's is generated


# ---------------------------------------------------------------- workload --
class Workload:
    def __init__(self, n, n_g=R18_N_G, d=0.01, dtype="f32", beta=1.25, stream="default",
                 seed=SEED):
        self.n, self.n_g, self.d, self.dtype, self.beta = n, n_g, d, dtype, beta
        self.stream, self.seed = stream, seed

    @property
    def default(self):
        return (self.n_g, self.d, self.dtype, self.beta, self.stream) == (
            R18_N_G, 0.01, "f32", 1.25, "default")

    def cfg_kw(self):
        # every parameter pinned (SURVEY.md §7 hard part 10)
        return dict(n=self.n, n_g=self.n_g, n_b=N_B, d=self.d, alpha=1.25, beta=self.beta,
                    gamma=0.02, blk_move=1, min_blk=2, eta=1.0, seed=self.seed)

    def segments(self):
        if self.stream == "skew":  # acceptance_main.cpp:107-111: 8 segments, 1.0/0.25
            base = self.n_g // 8
            segs = [(base, 1.0 if i % 2 == 0 else 0.25) for i in range(8)]
            segs[-1] = (self.n_g - base * 7, segs[-1][1])
            return segs
        return None  # run_config.cpp:248-260: the default four-segment stream

    def name(self):
        if self.default:
            return "configs[1]: ResNet-18-sized gradient, partitioned sparsify+sync"
        if self.n_g == R18_N_G:
            return "configs[1] variant (ResNet-18-sized gradient)"
        if self.n_g == 6_200_000:
            return "configs[2]: GoogLeNet-sized gradient"
        if self.n_g == 11_300_000:
            return "configs[3]: SENet-18-sized gradient"
        return "configs[4]: scaling-sweep cell"

    def metric(self):
        return (f"sparsify+sync ms/iter (ExDyna step, n_g={self.n_g}, d={self.d}"
                + ("" if self.dtype == "f32" else f", {self.dtype}")
                + ("" if self.beta == 1.25 else f", beta={self.beta}")
                + ("" if self.stream == "default" else f", {self.stream} stream") + ")")

    def config(self):
        return {"workload": self.name(), "n_g": self.n_g, "d": self.d,
                "k": round(self.d * self.n_g), "n_b": N_B, "workers": self.n,
                "alpha": 1.25, "beta": self.beta, "gamma": 0.02, "min_blk": 2, "blk_move": 1,
                "delta0": "auto (t=0 quantile)",
                "stream": ("default 4-segment Laplace" if self.stream == "default"
                           else "skew: 8 segments alternating 1.0/0.25") + f", seed {self.seed}",
                "l2": "flushed before every timed step (2x L2 buffer written, then read back)",
                "parallelism": f"dp{self.n}", "sync": "single GPU" if self.n == 1 else None}

    def esize(self):
        return 8 if self.dtype == "f64" else 4


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


def host_mem_available():
    try:
        for line in open("/proc/meminfo"):
            if line.startswith("MemAvailable:"):
                return int(line.split()[1]) * 1024
    except OSError:
        pass
    return None


def cpu_run(kind, wl, grad_fn, steps=50, warmup=5, budget_s=20.0, lean=False):
    """Time one CPU implementation of Engine::step() on this host.

    kind "reference": the unmodified reference (oracle/_ref), fp64, n worker
    threads (engine.cpp:90-117); kind "port": the fp32 C restatement
    (oracle/liboracle.so), the bit-exact checker of the fp32 GPU path.
    grad_fn(t) returns the n host gradients of step t (fresh every step, like
    the GPU run); they are handed to the replay GradientSource of ref_shim.cpp
    before the step's clock starts. Median ms/iter over up to `steps` steps
    after `warmup`, fewer when the timed steps would overrun
    `budget_s`. Returns (median, times, records)."""
    import numpy as np
    from oracle import oracle as O
    cfg = O.make_config(**wl.cfg_kw())
    n = wl.n
    if kind == "reference":
        if not O.ref_available():
            raise RuntimeError("oracle/_ref/libsparsim_ref.so not built")
        opt = O.make_options(verify_replication=0 if lean else 1, record_loss=0 if lean else 1)
        eng = O.RefEngine(cfg, opt, pool=n)  # step t, rank r reads slot (t*n + r) % n = r

        def step(gs):
            for r, g in enumerate(gs):
                eng.set_slot(r, g)
            a = time.perf_counter()
            rec = eng.step()
            return rec, time.perf_counter() - a
    else:
        eng = O.OracleEngine(cfg, np.float32, verify_replication=False)

        def step(gs):
            gs = [np.ascontiguousarray(g, dtype=np.float32) for g in gs]
            a = time.perf_counter()
            rec = eng.step(gs)
            return rec, time.perf_counter() - a
    recs, times = [], []
    spent = 0.0
    for t in range(warmup + steps):
        rec, dt = step(grad_fn(t))
        recs.append(rec)
        if t >= warmup:
            times.append(dt * 1e3)
            spent += dt
            if spent > budget_s and len(times) >= 3:
                break
    return statistics.median(times), times, recs


def reference_grad_fn(wl):
    """Gradients for the reference arm from the reference's own generator
    (workloads.cpp:62-85 through ref_shim), rounded to fp32 like the GPU's; the
    n ranks of a step are generated on parallel host threads (untimed)."""
    import numpy as np
    from concurrent.futures import ThreadPoolExecutor
    from oracle import oracle as O
    spec = O.stream_spec(wl.n_g, wl.segments(), seed=wl.seed)
    pool = ThreadPoolExecutor(max_workers=max(1, min(wl.n, os.cpu_count() or 1)))

    def one(tr):
        return O.synthetic_gradient_ref(spec, tr[0], tr[1]).astype(np.float32)

    return lambda t: list(pool.map(one, [(t, r) for r in range(wl.n)]))


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    wl = workload_of(args)
    n = wl.n
    try:
        warmup = max(5, args.warmup)
        ms, times, _ = cpu_run("reference", wl, reference_grad_fn(wl), steps=max(50, args.steps),
                               warmup=warmup, budget_s=60.0)
    except Exception as e:  # the reference is always buildable here; report why not
        print(json.dumps({"impl": "reference", "unavailable": str(e)}))
        return 0
    cores = n  # sparsim runs n-1 worker threads + the caller (engine.cpp:90-117)
    line = {
        "metric": wl.metric(), "value": ms, "unit": UNIT, "n_gpus": n, "steps": len(times),
        "warmup": warmup, "ms_per_step": ms, "higher_is_better": False, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
        "config": wl.config(),
        "cpu_baseline": {"value": ms, "unit": UNIT, "cores": cores, "kind": "reference",
                         "sample": f"median of {len(times)} full Engine::step() calls with {n} "
                                   f"simulated workers after {warmup} warm-up steps (t=0 "
                                   f"quantile included in the warm-up); as shipped: "
                                   f"verify_replication on, worker threads on; a fresh "
                                   f"fp32-rounded gradient per rank per step from the "
                                   f"reference's generator (replay source, generation "
                                   f"untimed); {host_cpu()}",
                         "mean": statistics.mean(times), "min": min(times), "max": max(times)},
        "e2e": {"value": ms, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


def cpu_baseline(wl, grad_fn, budget_s):
    """BASELINE.md §3 at N = 1: as shipped, lean, and the fp32 restatement, on
    the GPU run's own gradients (copied to the host)."""
    need = 6 * wl.n_g * 8  # x, e, acc, slots of the fp64 reference (+ verify snapshot)
    avail = host_mem_available()
    if avail is not None and avail < 1.5 * need:
        return {"value": None, "unit": UNIT, "cores": 1, "kind": "reference",
                "sample": f"skipped: host MemAvailable {avail / 2**30:.1f} GiB < "
                          f"1.5 x {need / 2**30:.1f} GiB for the fp64 reference at n_g={wl.n_g}"}
    big = wl.n_g > 50_000_000
    warm = 2 if big else 5
    out = {}
    for key, kind, lean in (("as_shipped", "reference", False), ("lean", "reference", True),
                            ("fp32_restatement", "port", False)):
        try:
            ms, times, recs = cpu_run(kind, wl, grad_fn, steps=50, warmup=warm,
                                      budget_s=budget_s, lean=lean)
            out[key] = {"median_ms": ms, "mean_ms": statistics.mean(times), "steps": len(times),
                        "warmup": warm,
                        "density_mean": statistics.mean(r.density for r in recs[warm:])}
        except Exception as e:
            out[key] = {"unavailable": str(e)}
    if wl.default and wl.n == 1:
        # configs[0]: the same gradient size with 2 simulated workers, the reference's own
        # CPU run (BASELINE.json configs[0]); the reference runs one thread per worker
        try:
            wl2 = Workload(2, n_g=wl.n_g, d=wl.d)
            ms, times, recs = cpu_run("reference", wl2, reference_grad_fn(wl2), steps=20,
                                      warmup=warm, budget_s=budget_s)
            out["configs0_n2_as_shipped"] = {"median_ms": ms, "mean_ms": statistics.mean(times),
                                             "steps": len(times), "warmup": warm, "cores": 2}
        except Exception as e:
            out["configs0_n2_as_shipped"] = {"unavailable": str(e)}
    v = out.get("as_shipped", {}).get("median_ms")
    return {"value": v, "unit": UNIT, "cores": wl.n, "kind": "reference",
            "sample": f"median over up to 50 Engine::step() calls (fewer when a step would "
                      f"overrun {budget_s:.0f} s) after {warm} warm-up steps of the unmodified "
                      f"reference (oracle/_ref, -O3 -ffp-contract=off) with {wl.n} worker "
                      f"thread(s), fed the GPU run's own gradient stream (device-generated, "
                      f"copied to the host before each step's clock starts; replay source); "
                      f"value = as shipped (verify_replication on); {host_cpu()}",
            "settings": out}


# ------------------------------------------------------------ ncu traffic ----
def ncu_path():
    p = shutil.which("ncu")
    if p:
        return p
    p = "/usr/local/cuda/bin/ncu"
    return p if os.path.exists(p) else None


def ncu_child(args):
    """Under ncu: t = 0 plus 3 fused steps with L2 flushed before each."""
    import torch
    from paper_2402_13781_b200 import sparsim as S
    wl = workload_of(args)
    torch.cuda.set_device(0)
    eng = S.Engine(S.SparsifierConfig(**wl.cfg_kw()), S.EngineOptions(dtype=wl.dtype), device=0)
    src = S.SyntheticStream(S.StreamSpec(n_g=wl.n_g, segments=wl.segments(), seed=wl.seed))
    td = torch.float64 if wl.dtype == "f64" else torch.float32
    buf = torch.empty(wl.n_g, dtype=td, device="cuda:0")
    for t in range(4):
        src.gradient(t, 0, buf, wl.dtype, eng.stream())
        S.flush_l2(0, eng.stream())
        eng.step([buf])
    return 0


def ncu_traffic(args, timeout=240):
    """DRAM bytes and duration per launch of K1 (stream_kernel, fused) and K2
    (finish_kernel), measured by ncu in a child process of this run (cold
    cache: ncu flushes caches before each profiled launch)."""
    ncu = ncu_path()
    if not ncu:
        return {"source": "unavailable: ncu not found"}
    cmd = [ncu, "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum",
           "--clock-control", "none", "--print-units", "base", "-k", "regex:stream_kernel|finish_kernel", "--csv",
           sys.executable, os.path.join(ROOT, "bench.py"), "--ncu-child",
           "--n_g", str(args.n_g), "--density", str(args.density), "--dtype", args.dtype,
           "--beta", str(args.beta), "--stream", args.stream]
    try:
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout)
    except Exception as e:
        return {"source": f"unavailable: {e}"}
    import csv
    import io
    rows = [l for l in r.stdout.splitlines() if l.startswith('"')]
    if not rows:
        return {"source": f"unavailable: ncu rc={r.returncode}: {r.stderr[-300:]}"}
    launches = {}
    try:
        return ncu_parse(csv.DictReader(io.StringIO("\n".join(rows))), launches)
    except Exception as e:
        return {"source": f"unavailable: ncu output not parsed: {e}"}


def ncu_parse(reader, launches):
    for row in reader:
        key = (row["ID"], row["Kernel Name"])
        d = launches.setdefault(key, {"name": row["Kernel Name"]})
        unit = row.get("Metric Unit", "")
        val = float(row["Metric Value"].replace(",", ""))
        scale = {"byte": 1, "B": 1, "Kbyte": 1e3, "KB": 1e3, "Mbyte": 1e6, "MB": 1e6,
                 "Gbyte": 1e9, "GB": 1e9, "nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6,
                 "us": 1e-6, "msecond": 1e-3, "ms": 1e-3, "second": 1.0, "s": 1.0}.get(unit)
        if scale is None:
            raise ValueError(f"ncu unit {unit!r} of {row['Metric Name']}")
        d[row["Metric Name"]] = val * scale
    order = sorted(launches, key=lambda k: int(k[0]))

    def last(pred):
        ks = [k for k in order if pred(launches[k]["name"])]
        return launches[ks[-1]] if ks else None

    k1 = last(lambda s: "stream_kernel" in s and ", 0," in s)  # MODE kFused
    k2 = last(lambda s: "finish_kernel" in s)
    out = {"source": "ncu in this run (bench.py --ncu-child; cold cache, serialised)",
           "launches_profiled": len(order)}
    for tag, d in (("k1", k1), ("k2", k2)):
        if d:
            rb = d.get("dram__bytes_read.sum", 0.0)
            wb = d.get("dram__bytes_write.sum", 0.0)
            out[tag] = {"kernel": d["name"][:120], "dram_read": rb, "dram_write": wb,
                        "dram_bytes": rb + wb, "duration_s": d.get("gpu__time_duration.sum")}
    return out


# ------------------------------------------------------------------ ours ----
def workload_of(args):
    n = args.gpus
    return Workload(n, n_g=args.n_g, d=args.density, dtype=args.dtype, beta=args.beta,
                    stream=args.stream)


def device_grad_fn(S, torch, wl, local, stream_ptr):
    """grad_fn for the CPU legs: the GPU run's own stream (device generator,
    step t, rank r), rounded to fp32 and copied to the host."""
    src = S.SyntheticStream(S.StreamSpec(n_g=wl.n_g, segments=wl.segments(), seed=wl.seed))
    buf = torch.empty(wl.n_g, dtype=torch.float32, device=f"cuda:{local}")

    def fn(t):
        out = []
        for r in range(wl.n):
            src.gradient(t, r, buf, "f32", stream_ptr)
            torch.cuda.synchronize()
            out.append(buf.cpu().numpy())
        return out
    return fn


def variant_run(S, torch, base_wl, local, dtype, beta, steps=400):
    """A fresh engine from t = 0 on the fp32-rounded device stream, timed per
    step like the main line (L2 flushed, CUDA events on the engine stream)."""
    wl = Workload(1, n_g=base_wl.n_g, d=base_wl.d, dtype=dtype, beta=beta)
    opt = S.EngineOptions(dtype=dtype, verify_replication=False, record_loss=False)
    eng = S.Engine(S.SparsifierConfig(**wl.cfg_kw()), opt, device=local)
    stream = torch.cuda.ExternalStream(eng.stream())
    src = S.SyntheticStream(S.StreamSpec(n_g=wl.n_g, seed=wl.seed))
    g32 = torch.empty(wl.n_g, dtype=torch.float32, device=f"cuda:{local}")
    buf = torch.empty(wl.n_g, dtype=torch.float64 if dtype == "f64" else torch.float32,
                      device=f"cuda:{local}")
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(steps)]
    for a_, b_ in ev:
        a_.record(stream)
        b_.record(stream)
    S.flush_l2(local, eng.stream())
    torch.cuda.synchronize()
    recs = []
    for t in range(steps):
        src.gradient(t, 0, g32, "f32", eng.stream())  # the same fp32 values the reference reads
        with torch.cuda.stream(stream):
            buf.copy_(g32)
        S.flush_l2(local, eng.stream())
        ev[t][0].record(stream)
        eng.step_async([buf])
        ev[t][1].record(stream)
        recs.append(eng.sync())
    ms = [a.elapsed_time(b) for a, b in ev]
    eng.close()
    return wl, ms, recs


def variants(S, torch, wl, local, budget_s, stream_ptr):
    """fp64 GPU path and beta = 1.05 at the default config, each with its
    density next to the reference's own on the same inputs."""
    out = []
    for dtype, beta in (("f64", 1.25), ("f32", 1.05)):
        vwl, ms, recs = variant_run(S, torch, wl, local, dtype, beta)
        steady = recs[len(recs) // 2:]  # the controller has settled (delta moves 2% a step)
        item = {"dtype": dtype, "beta": beta, "steps": len(ms),
                "step_ms_median_t_ge_5": statistics.median(ms[5:]),
                "step_ms_mean_t_ge_5": statistics.mean(ms[5:]),
                "density_mean_steady": statistics.mean(r.density for r in steady),
                "density_over_d_steady": statistics.mean(r.density for r in steady) / wl.d,
                "steady_window": [steady[0].t, steady[-1].t]}
        try:
            # the reference on the same inputs for the first 60 steps: its
            # timing, and its density / records next to the GPU's
            rms, rtimes, rrecs = cpu_run("reference", vwl, device_grad_fn(S, torch, vwl, local,
                                                                          stream_ptr),
                                         steps=55, warmup=5, budget_s=budget_s)
            m = min(len(rrecs), len(recs))
            item["reference"] = {
                "median_ms": rms, "steps_timed": len(rtimes), "steps": m,
                "density_mean_t_ge_5": statistics.mean(r.density for r in rrecs[5:m]),
                "density_mean_t_ge_5_gpu_same_steps": statistics.mean(r.density for r in recs[5:m])}
            if dtype == "f64":  # bit-exact with the reference: k', delta, k_rank agree
                item["records_identical_to_reference"] = all(
                    (a.k_prime, a.delta, a.k_rank[0]) == (b.k_prime, b.delta, b.k_rank[0])
                    for a, b in zip(recs[:m], rrecs[:m]))
        except Exception as e:
            item["reference"] = {"unavailable": str(e)}
        out.append(item)
    return out


def pin_to_gpu_cpus(index):
    """Run this process on the CPUs local to GPU `index` (NVML affinity), so the
    pinned host buffers of the e2e leg are first touched on the GPU's NUMA node."""
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(index)
        words = pynvml.nvmlDeviceGetCpuAffinity(h, (os.cpu_count() + 63) // 64)
        cpus = {w * 64 + b for w, m in enumerate(words) for b in range(64) if (m >> b) & 1}
        cpus &= set(range(os.cpu_count()))
        if cpus:
            os.sched_setaffinity(0, cpus)
            return sorted(cpus)
    except Exception:
        pass
    return None


def run_ours(args):
    import numpy as np
    import torch

    from paper_2402_13781_b200 import sparsim as S

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    wl = workload_of(args)
    n = wl.n
    if world != n:
        raise SystemExit(f"--gpus {n} but WORLD_SIZE={world}; launch N>1 with torchrun")
    cpus = pin_to_gpu_cpus(local)
    torch.cuda.set_device(local)
    dist = None
    if n > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")  # control plane only; the data path is NCCL in C++
    N_G = wl.n_g
    td = torch.float64 if wl.dtype == "f64" else torch.float32
    opt = S.EngineOptions(dtype=wl.dtype, profile_kernels=False, verify_replication=False,
                          record_loss=False, sync=args.sync)
    if n == 1:
        eng = S.Engine(S.SparsifierConfig(**wl.cfg_kw()), opt, device=local)
    else:
        obj = [S.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        eng = S.Engine.rank(S.SparsifierConfig(**wl.cfg_kw()), opt, rank, local, obj[0])
    stream = torch.cuda.ExternalStream(eng.stream())
    src = S.SyntheticStream(S.StreamSpec(n_g=N_G, segments=wl.segments(), seed=wl.seed))
    bufs = [torch.empty(N_G, dtype=td, device=f"cuda:{local}") for _ in range(POOL)]
    for i, b in enumerate(bufs):
        src.gradient(i, rank, b, wl.dtype, eng.stream())
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
            src.gradient(i, rank, bufs[i % POOL], wl.dtype, eng.stream())  # fresh g_t (untimed)
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
        src.gradient(i, rank, bufs[i % POOL], wl.dtype, eng.stream())
        eng.step_async([bufs[i % POOL]])
        i += 1

    recs = []
    for k in range(args.steps):
        src.gradient(i + k, rank, bufs[(i + k) % POOL], wl.dtype, eng.stream())  # untimed
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
        src.gradient(i + k, rank, bufs[(i + k) % POOL], wl.dtype, eng.stream())
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
        h = torch.empty(N_G, dtype=td, pin_memory=True)
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
    sync_mode = eng.sync_mode()

    if rank != 0:
        eng.close()
        if dist:
            dist.barrier()
        return 0

    # roofline of the dominant kernel (fused accumulate+select+compact)
    kp = statistics.mean(r.k_prime for r in recs)
    k_own = statistics.mean(r.k_rank[0] for r in recs)
    es = wl.esize()
    # K1's algorithmic bytes: read g, read e, write e over the full
    # vector (engine.cpp:135-141) + the staged (index, value) pairs of the own
    # selection (selector.cpp:38-40)
    alg_bytes = 3 * es * N_G + (4 + es) * k_own
    achieved = alg_bytes / (sel_ms * 1e-3) / 1e9
    peak, peak_src = peaks()
    eng.close()
    del bufs
    torch.cuda.empty_cache()

    traffic = None
    ncu = None
    if n == 1 and args.traffic == "ncu":
        ncu = ncu_traffic(args)
        if "k1" in ncu:
            traffic = ncu["k1"]["dram_bytes"]
            d = ncu["k1"]["duration_s"]
            ncu["k1"]["dram_gbs"] = traffic / d / 1e9 if d else None
            ncu["k1"]["dram_frac"] = traffic / d / 1e9 / peak if d else None
            ncu["k1"]["algorithmic_gbs"] = alg_bytes / d / 1e9 if d else None
            ncu["k1"]["algorithmic_frac"] = alg_bytes / d / 1e9 / peak if d else None
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": traffic,
            "kernel": f"stream_kernel<{'double' if es == 8 else 'float'},kFused> "
                      "(K1: accumulate + select + stage)",
            "kernel_ms": sel_ms, "finish_kernel_ms": fin_ms,
            "algorithmic_bytes_per_launch": alg_bytes,
            "algorithmic_bytes_formula": f"3*{es}*n_g + ({4 + es})*k_i (k_i = own selection)",
            "peak_source": peak_src, "share_of_step": sel_ms / ms, "ncu": ncu}

    cpu = None
    var = None
    if n == 1 and args.cpu != "none":
        cpu = cpu_baseline(wl, device_grad_fn(S, torch, wl, local, 0), budget_s=args.cpu_budget)
        if wl.default and args.variants:
            var = variants(S, torch, wl, local, args.cpu_budget, 0)

    # sync stage over NVLink (push-reduce): algorithmic bytes each GPU stores into
    # its peers' inboxes per step, against the exchange kernel's event time
    nvlink = None
    if n > 1 and sync_mode == "p2p":
        tiles_own = (N_G / n) / (4096.0 if es == 4 else 2048.0)
        holder = (n >= 4) if "EXD_HOLDER_SUM" not in os.environ else os.environ["EXD_HOLDER_SUM"] == "1"
        words = (kp - k_own) + (n - 1) * k_own if holder else (n - 1) * kp  # contribution/sum words out
        out_b = (n - 1) * (8 * k_own + 72 * tiles_own) + 8 * (es // 4) * words
        nvlink = {"bytes_out_per_gpu_per_step": out_b, "sync_kernel_ms": fin_ms,
                  "achieved_gbs": out_b / (fin_ms * 1e-3) / 1e9, "peak_gbs": 770.0,
                  "peak_source": "measured peer copy per direction (B200_PROFILING.md; 900 "
                                 "nominal); the protocol's posted word stores reach 710 GB/s "
                                 "alone (profiles/nvlink_word_ceiling_r02.txt)",
                  "frac": out_b / (fin_ms * 1e-3) / 1e9 / 770.0,
                  "note": "algorithmic bytes / event time; bytes = staged-index and count "
                          "words pushed by the stream kernel + contribution words "
                          "(to every peer, or to the holder and sums back for n >= 4)",
                  "holder_sum": holder}
    cfg_line = wl.config()
    if n > 1:
        cfg_line["sync"] = {
            "p2p": "NVLink peer memory, push-reduce (lists pushed during the stream, "
                   "everything as {payload, epoch} words; no handshake, no host wait)",
            "p2p-pull": "NVLink peer memory, pull-reduce (lists pushed, contributions pulled)",
            "nccl": "NCCL all-gather/all-reduce + one host wait"}[sync_mode]
    line = {
        "metric": wl.metric(), "value": ms, "unit": UNIT, "n_gpus": n, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False, "scaling": "weak",
        "vs_baseline": None, "dtype": wl.dtype, "data": "synthetic", "config": cfg_line,
        "selection_hbm_gbs": achieved,
        "roofline": roof,
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_ms, "unit": UNIT, "h2d_bytes_per_step": es * N_G * n,
                "d2h_bytes_per_step": C.sizeof(A.exd_record) * n,
                "h2d_gbs": es * N_G / (e2e_ms * 1e-3) / 1e9,
                "host_cpus": f"{len(cpus)} GPU-local CPUs (NVML affinity)" if cpus else "unpinned"},
        "gpu_launches": launches,
        "nvlink": nvlink,
        "clocks": clk,
        "records": {"k_prime_mean": kp, "f_t_mean": statistics.mean(r.f_t for r in recs),
                    "density_mean": statistics.mean(r.density for r in recs),
                    "density_over_d": statistics.mean(r.density for r in recs) / wl.d,
                    "t_last": recs[-1].t},
        "step_ms_min": min(step_ms), "step_ms_median": statistics.median(step_ms),
        "step_ms_p90": sorted(step_ms)[int(0.9 * (len(step_ms) - 1))], "step_ms_max": max(step_ms),
    }
    if var is not None:
        line["variants"] = var
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
    ap.add_argument("--n_g", type=int, default=R18_N_G)
    ap.add_argument("--density", type=float, default=0.01)
    ap.add_argument("--dtype", default="f32", choices=["f32", "f64"])
    ap.add_argument("--beta", type=float, default=1.25)
    ap.add_argument("--stream", default="default", choices=["default", "skew"])
    ap.add_argument("--cpu", default="auto", choices=["auto", "none"],
                    help="N = 1: time the CPU reference on this host (cpu_baseline)")
    ap.add_argument("--cpu-budget", type=float, default=20.0,
                    help="seconds of timed CPU steps per setting")
    ap.add_argument("--traffic", default="ncu", choices=["ncu", "none"],
                    help="N = 1: K1's DRAM bytes by ncu in a child process of this run")
    ap.add_argument("--no-variants", dest="variants", action="store_false")
    ap.add_argument("--ncu-child", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.ncu_child:
        return ncu_child(args)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
