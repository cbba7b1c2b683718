"""oracle/oracle.py — TEST INFRASTRUCTURE ONLY.

ctypes bindings for the two checkers:
  * liboracle.so            C restatement of the reference step (exdyna_oracle.c)
  * _ref/libsparsim_ref.so  the unmodified reference library + ref_shim.cpp
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs import this module. The product package never does.
"""
import ctypes as C
import os

import numpy as np

from paper_2402_13781_b200 import _abi as A

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libsparsim_ref.so")

P = C.c_void_p
PI64 = C.POINTER(C.c_int64)
PI32 = C.POINTER(C.c_int32)
PD = C.POINTER(C.c_double)


def build():
    """Compile the oracle (and oracle/_ref when /root/reference is present)."""
    import subprocess
    subprocess.run(["make", "-s", "-C", HERE], check=True)


_orc = None
_ref = None


def orc():
    global _orc
    if _orc is None:
        if not os.path.exists(ORACLE_SO):
            build()
        L = C.CDLL(ORACLE_SO)
        L.orc_last_error.restype = C.c_char_p
        L.orc_validate.argtypes = [C.POINTER(A.exd_config), C.POINTER(A.exd_config)]
        L.orc_build_topology.argtypes = [C.c_int64, C.c_int64, C.c_int32, C.c_int64,
                                         C.POINTER(A.exd_topology), C.c_char_p, C.c_size_t]
        L.orc_partition_range.argtypes = [C.POINTER(A.exd_topology), C.c_int32, C.c_int64, PI64, PI64]
        L.orc_rotate.argtypes = [PI64, C.c_int64, C.c_int32, PI64]
        L.orc_adjust.argtypes = [C.POINTER(A.exd_topology), PI64, C.c_double, C.c_int64,
                                 C.c_int64, C.c_int64, PI32, PI32]
        L.orc_allocate.argtypes = [C.POINTER(A.exd_topology), C.c_int64, C.c_int32, C.c_int64,
                                   PI32, PI64, PI64]
        L.orc_scale_threshold.restype = C.c_double
        L.orc_scale_threshold.argtypes = [C.c_int64, C.c_int64, C.c_double, C.c_double, C.c_double]
        L.orc_initial_threshold.argtypes = [PD, C.c_int64, C.c_double, PD]
        L.orc_gather_stats.argtypes = [PI64, C.c_int32, C.POINTER(A.exd_gather_stats)]
        L.orc_synthetic_gradient.argtypes = [C.POINTER(A.exd_stream_spec), C.c_int64, C.c_int32, PD]
        for suf in ("f32", "f64"):
            getattr(L, f"orc_create_{suf}").restype = P
            getattr(L, f"orc_create_{suf}").argtypes = [C.POINTER(A.exd_config), C.c_int, C.c_int]
            getattr(L, f"orc_destroy_{suf}").argtypes = [P]
            getattr(L, f"orc_set_grad_{suf}").argtypes = [P, C.c_int, P]
            getattr(L, f"orc_step_{suf}").argtypes = [P, C.POINTER(A.exd_record)]
            for nm in ("orc_x", "orc_e", "orc_x_mut"):
                getattr(L, f"{nm}_{suf}").restype = P
                getattr(L, f"{nm}_{suf}").argtypes = [P, C.c_int]
            getattr(L, f"orc_sum_{suf}").restype = P
            getattr(L, f"orc_sum_{suf}").argtypes = [P]
            getattr(L, f"orc_union_{suf}").restype = C.c_int64
            getattr(L, f"orc_union_{suf}").argtypes = [P, C.POINTER(PI64)]
            getattr(L, f"orc_selection_{suf}").restype = C.c_int64
            getattr(L, f"orc_selection_{suf}").argtypes = [P, C.c_int, C.POINTER(PI64)]
            getattr(L, f"orc_state_{suf}").argtypes = [P, C.c_int, C.POINTER(A.exd_worker_state)]
            getattr(L, f"orc_block_counts_{suf}").argtypes = [P, C.c_int, PI32]
        _orc = L
    return _orc


def ref_available():
    return os.path.exists(REF_SO)


def ref():
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            build()
        if not os.path.exists(REF_SO):
            raise RuntimeError("oracle/_ref/libsparsim_ref.so is not built "
                               "(reference tree absent and no prebuilt copy)")
        L = C.CDLL(REF_SO)
        L.ref_last_error.restype = C.c_char_p
        L.ref_validate.argtypes = [C.POINTER(A.exd_config), C.POINTER(A.exd_config)]
        L.ref_build_topology.argtypes = [C.c_int64, C.c_int64, C.c_int32, C.c_int64,
                                         C.POINTER(A.exd_topology), C.c_char_p, C.c_size_t]
        L.ref_partition_range.argtypes = [C.POINTER(A.exd_topology), C.c_int32, C.c_int64, PI64, PI64]
        L.ref_rotate.argtypes = [PI64, C.c_int64, C.c_int32, PI64]
        L.ref_adjust.argtypes = [C.POINTER(A.exd_topology), PI64, C.c_double, C.c_int64,
                                 C.c_int64, C.c_int64, PI32, PI32]
        L.ref_allocate.argtypes = [C.POINTER(A.exd_topology), C.c_int64, C.c_int32, C.c_int64,
                                   PI32, PI64, PI64]
        L.ref_scale_threshold.restype = C.c_double
        L.ref_scale_threshold.argtypes = [C.c_int64, C.c_int64, C.c_double, C.c_double, C.c_double]
        L.ref_initial_threshold.argtypes = [PD, C.c_int64, C.c_double, PD]
        L.ref_all_gather.argtypes = [PI64, PI64, C.c_int32, C.POINTER(A.exd_gather_stats),
                                     PI64, PI64, PI64]
        L.ref_topk_select.argtypes = [PD, C.c_int64, C.c_int64, PI64]
        L.ref_hard_threshold_select.argtypes = [PD, C.c_int64, C.c_double, PI64, PI64]
        L.ref_synthetic_gradient.argtypes = [C.POINTER(A.exd_stream_spec), C.c_int64, C.c_int32, PD]
        L.ref_engine_create.restype = P
        L.ref_engine_create.argtypes = [C.POINTER(A.exd_config), C.POINTER(A.exd_options), C.c_int32]
        L.ref_engine_destroy.argtypes = [P]
        L.ref_engine_set_slot_f64.argtypes = [P, C.c_int32, PD]
        L.ref_engine_set_slot_f32.argtypes = [P, C.c_int32, C.POINTER(C.c_float)]
        L.ref_engine_step.argtypes = [P, C.POINTER(A.exd_record), C.c_int32]
        L.ref_engine_iteration.restype = C.c_int64
        L.ref_engine_iteration.argtypes = [P]
        L.ref_engine_get_vec.argtypes = [P, C.c_int32, C.c_int32, PD]
        L.ref_engine_poke_x.argtypes = [P, C.c_int32, C.c_int64, C.c_double]
        L.ref_engine_get_state.argtypes = [P, C.c_int32, C.POINTER(A.exd_worker_state)]
        L.ref_engine_last_selection.restype = C.c_int64
        L.ref_engine_last_selection.argtypes = [P, C.c_int32, PI64]
        L.ref_engine_last_union.restype = C.c_int64
        L.ref_engine_last_union.argtypes = [P, PI64]
        L.ref_format_csv.restype = C.c_int64
        L.ref_format_csv.argtypes = [C.POINTER(A.exd_record), C.c_int64, C.c_char_p, C.c_int64]
        L.ref_summarize.argtypes = [C.POINTER(A.exd_record), C.c_int64, PD, PI64]
        _ref = L
    return _ref


def records_array(recs):
    """list of exd_record (or record dicts) -> ctypes array"""
    arr = (A.exd_record * max(1, len(recs)))()
    for i, r in enumerate(recs):
        if isinstance(r, A.exd_record):
            arr[i] = r
            continue
        c = arr[i]
        for f in A.RECORD_FIELDS:
            setattr(c, f, r[f])
        c.has_loss, c.loss = (1, r["loss"]) if r.get("loss") is not None else (0, 0.0)
        c.n = len(r["k_rank"])
        for j, k in enumerate(r["k_rank"]):
            c.k_rank[j] = k
    return arr


def ref_format_csv(recs):
    arr = records_array(recs)
    n = ref().ref_format_csv(arr, len(recs), None, 0)
    buf = C.create_string_buffer(n + 1)
    ref().ref_format_csv(arr, len(recs), buf, n + 1)
    return buf.value.decode()


class CheckError(Exception):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


def _ptr(a, ctype):
    return a.ctypes.data_as(C.POINTER(ctype))


def make_config(**kw):
    """exd_config with the reference's SparsifierConfig defaults (config.hpp:28-45)."""
    c = A.exd_config()
    c.n, c.n_g, c.n_b, c.d = 4, 1_000_000, 256, 0.001
    c.alpha, c.beta, c.gamma = 1.25, 1.25, 0.02
    c.blk_move, c.min_blk, c.eta, c.seed = 1, 2, 1.0, 42
    for k, v in kw.items():
        if k == "delta0":
            if v is not None:
                c.has_delta0, c.delta0 = 1, v
        elif k == "max_density_cap":
            if v is not None:
                c.has_max_density_cap, c.max_density_cap = 1, v
        else:
            setattr(c, k, v)
    return c


def make_options(**kw):
    o = A.exd_options()
    o.sparsifier = A.EXD_SPARSIFIER_EXDYNA
    o.parallel_workers, o.verify_replication, o.record_loss = 1, 1, 1
    for k, v in kw.items():
        setattr(o, k, v)
    return o


def stream_spec(n_g, segments=None, seed=42, distribution=0, decay=1.0,
                decay_step=None, decay_step_factor=0.1):
    """StreamSpec (workloads.hpp:121-129). segments=None: the default
    four-segment stream of run_config.cpp:248-260."""
    if segments is None:
        q = n_g // 4
        segments = ([(q, 1.0), (q, 0.5), (q, 0.25), (n_g - 3 * q, 0.125)]
                    if q > 0 else [(n_g, 1.0)])
    s = A.exd_stream_spec()
    s.n_g, s.nseg, s.distribution = n_g, len(segments), distribution
    for i, (ln, sc) in enumerate(segments):
        s.seg_length[i], s.seg_scale[i] = ln, sc
    s.decay, s.decay_step_factor, s.seed = decay, decay_step_factor, seed
    if decay_step is not None:
        s.has_decay_step, s.decay_step = 1, decay_step
    return s


def skew_segments(n_g, nseg=8, hot=1.0, cold=0.25):
    """acceptance_main.cpp:98-113 skew layout: equal segments alternating hot/cold."""
    base = n_g // nseg
    segs = [(base, hot if i % 2 == 0 else cold) for i in range(nseg)]
    segs[-1] = (n_g - base * (nseg - 1), segs[-1][1])
    return segs


def synthetic_gradient_orc(spec, t, rank):
    out = np.empty(spec.n_g, dtype=np.float64)
    orc().orc_synthetic_gradient(C.byref(spec), t, rank, _ptr(out, C.c_double))
    return out


def synthetic_gradient_ref(spec, t, rank):
    out = np.empty(spec.n_g, dtype=np.float64)
    rc = ref().ref_synthetic_gradient(C.byref(spec), t, rank, _ptr(out, C.c_double))
    if rc:
        raise CheckError(rc, ref().ref_last_error().decode())
    return out


# ---- baseline sparsifiers: numpy restatement -----------
def topk_select_np(acc, k):
    """baselines.cpp:26-41: the k largest |acc| under the total order
    (|a| desc, index asc) of its nth_element comparator (:33-37), ascending."""
    n = acc.shape[0]
    if k < 1 or k > n:
        raise ValueError("topk_select: k out of range")
    mag = np.abs(acc.astype(np.float64))
    order = np.lexsort((np.arange(n), -mag))
    return np.sort(order[:k]).astype(np.int64)


def hard_threshold_select_np(acc, fixed_delta):
    """baselines.cpp:43-46 -> select_indices over [0, n) (selector.cpp:35-42):
    ascending {j : |acc[j]| >= delta}, compared in fp64."""
    return np.flatnonzero(np.abs(acc.astype(np.float64)) >= fixed_delta).astype(np.int64)


def ref_topk_select(acc, k):
    """The unmodified reference's topk_select on fp64 acc."""
    a = np.ascontiguousarray(acc, dtype=np.float64)
    out = np.zeros(max(k, 1), np.int64)
    rc = ref().ref_topk_select(_ptr(a, C.c_double), a.shape[0], k, _ptr(out, C.c_int64))
    if rc:
        raise CheckError(rc, ref().ref_last_error().decode())
    return out[:k]


def ref_hard_threshold_select(acc, fixed_delta):
    a = np.ascontiguousarray(acc, dtype=np.float64)
    out = np.zeros(max(a.shape[0], 1), np.int64)
    cnt = C.c_int64()
    ref().ref_hard_threshold_select(_ptr(a, C.c_double), a.shape[0], fixed_delta,
                                    _ptr(out, C.c_int64), C.byref(cnt))
    return out[:cnt.value]


class OracleEngine:
    """The C restatement's engine (T = float32 or float64)."""

    def __init__(self, cfg, dtype=np.float32, static_partitions=False, verify_replication=True):
        self.L = orc()
        self.suf = "f32" if np.dtype(dtype) == np.float32 else "f64"
        self.dtype = np.dtype(dtype)
        self.h = getattr(self.L, f"orc_create_{self.suf}")(C.byref(cfg), int(static_partitions),
                                                          int(verify_replication))
        if not self.h:
            raise CheckError(A.EXD_EINVAL, self.L.orc_last_error().decode())
        v = A.exd_config()
        self.L.orc_validate(C.byref(cfg), C.byref(v))
        self.cfg = v
        self.n, self.n_g = v.n, v.n_g
        self._grads = [None] * self.n

    def __del__(self):
        if getattr(self, "h", None):
            getattr(self.L, f"orc_destroy_{self.suf}")(self.h)
            self.h = None

    def _f(self, name):
        return getattr(self.L, f"{name}_{self.suf}")

    def set_grad(self, r, g):
        g = np.ascontiguousarray(g, dtype=self.dtype)
        self._grads[r] = g
        self._f("orc_set_grad")(self.h, r, g.ctypes.data)

    def step(self, grads=None):
        if grads is not None:
            for r, g in enumerate(grads):
                self.set_grad(r, g)
        rec = A.exd_record()
        rc = self._f("orc_step")(self.h, C.byref(rec))
        if rc:
            raise CheckError(rc, self.L.orc_last_error().decode())
        return rec

    def _vec(self, name, r):
        p = self._f(name)(self.h, r)
        ct = C.c_float if self.suf == "f32" else C.c_double
        return np.ctypeslib.as_array(C.cast(p, C.POINTER(ct)), shape=(self.n_g,)).copy()

    def x(self, r=0):
        return self._vec("orc_x", r)

    def e(self, r=0):
        return self._vec("orc_e", r)

    def poke_x(self, r, j, v):
        p = self._f("orc_x_mut")(self.h, r)
        ct = C.c_float if self.suf == "f32" else C.c_double
        C.cast(p, C.POINTER(ct))[j] = v

    def union(self):
        p = PI64()
        n = self._f("orc_union")(self.h, C.byref(p))
        return np.ctypeslib.as_array(p, shape=(n,)).copy() if n else np.zeros(0, np.int64)

    def selection(self, r):
        p = PI64()
        n = self._f("orc_selection")(self.h, r, C.byref(p))
        return np.ctypeslib.as_array(p, shape=(n,)).copy() if n else np.zeros(0, np.int64)

    def sum(self):
        u = len(self.union())
        p = self._f("orc_sum")(self.h)
        ct = C.c_float if self.suf == "f32" else C.c_double
        return np.ctypeslib.as_array(C.cast(p, C.POINTER(ct)), shape=(u,)).copy() if u else np.zeros(0, self.dtype)

    def state(self, r):
        s = A.exd_worker_state()
        self._f("orc_state")(self.h, r, C.byref(s))
        return s

    def block_counts(self, r):
        out = np.zeros(self.cfg.n_b, dtype=np.int32)
        self._f("orc_block_counts")(self.h, r, _ptr(out, C.c_int32))
        return out


class RefEngine:
    """sparsim::Engine (unmodified) fed by the replay source in ref_shim.cpp."""

    def __init__(self, cfg, opt=None, pool=None):
        self.L = ref()
        opt = opt or make_options()
        self.n, self.n_g = cfg.n, cfg.n_g
        self.pool = pool or cfg.n
        self.h = self.L.ref_engine_create(C.byref(cfg), C.byref(opt), self.pool)
        if not self.h:
            raise CheckError(A.EXD_EINVAL, self.L.ref_last_error().decode())

    def __del__(self):
        if getattr(self, "h", None):
            self.L.ref_engine_destroy(self.h)
            self.h = None

    def set_slot(self, slot, g):
        if g.dtype == np.float32:
            g = np.ascontiguousarray(g)
            self.L.ref_engine_set_slot_f32(self.h, slot, _ptr(g, C.c_float))
        else:
            g = np.ascontiguousarray(g, dtype=np.float64)
            self.L.ref_engine_set_slot_f64(self.h, slot, _ptr(g, C.c_double))

    def iteration(self):
        return self.L.ref_engine_iteration(self.h)

    def step(self, grads=None, capture=False):
        """grads: per-rank vectors for THIS step (FixedSource semantics)."""
        if grads is not None:
            t = self.iteration()
            for r, g in enumerate(grads):
                self.set_slot((t * self.n + r) % self.pool, g)
        rec = A.exd_record()
        rc = self.L.ref_engine_step(self.h, C.byref(rec), int(capture))
        if rc:
            raise CheckError(rc, self.L.ref_last_error().decode())
        return rec

    def vec(self, r, which):
        out = np.empty(self.n_g, dtype=np.float64)
        self.L.ref_engine_get_vec(self.h, r, which, _ptr(out, C.c_double))
        return out

    def x(self, r=0):
        return self.vec(r, A.EXD_VEC_X)

    def e(self, r=0):
        return self.vec(r, A.EXD_VEC_E)

    def poke_x(self, r, j, v):
        self.L.ref_engine_poke_x(self.h, r, j, v)

    def state(self, r):
        s = A.exd_worker_state()
        self.L.ref_engine_get_state(self.h, r, C.byref(s))
        return s

    def selection(self, r):
        n = self.L.ref_engine_last_selection(self.h, r, None)
        out = np.empty(n, dtype=np.int64)
        self.L.ref_engine_last_selection(self.h, r, _ptr(out, C.c_int64))
        return out

    def union(self):
        n = self.L.ref_engine_last_union(self.h, None)
        out = np.empty(n, dtype=np.int64)
        self.L.ref_engine_last_union(self.h, _ptr(out, C.c_int64))
        return out


# ---- Engine runs of the baseline sparsifiers -----------
class BaselineOracle:
    """numpy restatement of sparsim::Engine::step for Top-k, CLT-k and hard
    threshold (engine.cpp:119-144 accumulate, :163-204 select, :274-350 step;
    all_gather / all_reduce_sum, collectives.cpp:22-70), T = float32 or
    float64. Pinned bit-exact against oracle/_ref in fp64
    (tests/test_baseline_oracle.py); the fp32 instance is the checker of the
    fp32 GPU path. Records are dicts with the IterationRecord field names."""

    KINDS = {"topk": 1, "cltk": 2, "hardthreshold": 3}

    def __init__(self, n, n_g, k, sparsifier, fixed_delta=0.0, eta=1.0, dtype=np.float32):
        self.n, self.n_g, self.k = n, n_g, k
        self.kind = sparsifier
        self.fixed_delta, self.eta = fixed_delta, eta
        self.T = np.dtype(dtype)
        self.x = [np.zeros(n_g, self.T) for _ in range(n)]
        self.e = [np.zeros(n_g, self.T) for _ in range(n)]
        self.k_t = [k // n] * n  # engine.cpp:77-78
        self.t = 0
        self.last_union = np.zeros(0, np.int64)
        self.last_sum = np.zeros(0, self.T)

    def step(self, grads):
        n, T = self.n, self.T
        norms = []
        for r in range(n):  # accumulate_phase, engine.cpp:134-141
            prev = self.e[r].astype(np.float64)
            norms.append(float(np.sqrt(np.dot(prev, prev))))
            acc = prev + self.eta * np.asarray(grads[r], dtype=np.float64)
            self.e[r] = acc.astype(T)
        sels = []
        leader = self.t % n  # cltk_leader, baselines.hpp:37-39
        for r in range(n):  # select_phase, engine.cpp:188-197
            if self.kind == "topk" or (self.kind == "cltk" and r == leader):
                sels.append(topk_select_np(self.e[r], self.k))
            elif self.kind == "hardthreshold":
                sels.append(hard_threshold_select_np(self.e[r], self.fixed_delta))
            else:
                sels.append(np.zeros(0, np.int64))
        k_rank = [len(s) for s in sels]
        total, m_t = sum(k_rank), max(k_rank)
        c_t = n * sum(m_t - c for c in k_rank)
        f_t = float(n) * float(m_t) / float(total) if total > 0 else 1.0
        union = np.unique(np.concatenate(sels)) if total else np.zeros(0, np.int64)
        dups = total - len(union)
        g = self.e[0][union].copy()  # contributions + rank-order sum (:310-319, :59-70)
        for r in range(1, n):
            g = (g + self.e[r][union]).astype(T)
        q = g.astype(np.float64) * (1.0 / n) if (n & (n - 1)) == 0 else g.astype(np.float64) / n
        for r in range(n):  # apply_phase, engine.cpp:206-219
            self.x[r][union] = (self.x[r][union].astype(np.float64) - q).astype(T)
            self.e[r][union] = 0
        self.k_t = list(k_rank)
        rec = {"t": self.t, "k_prime": total, "density": total / self.n_g,
               "eps": abs(self.k - total) / self.n_g, "m_t": m_t, "c_t": c_t, "f_t": f_t,
               "global_err": sum(norms) / n,
               "delta": self.fixed_delta if self.kind == "hardthreshold" else 0.0,
               "duplicates": dups, "union_count": len(union), "k_rank": k_rank,
               "adjust_moves": 0, "adjust_skips": 0, "cap_hits": 0,
               "idle_workers": n - 1 if self.kind == "cltk" else 0}
        self.last_union, self.last_sum = union, g
        self.t += 1
        return rec
