"""Host-side mirror of the reference's sparsifier API (sparsim, proj/include/sparsim).

Same names, argument meaning and error behaviour as the C++ reference, bound to
the B200 library through the C ABI of include/exdyna.h:

    SparsifierConfig / validate          config.hpp:28-45, config.cpp:28-51
    build_topology / partition_range     partition.hpp:25-44, partition.cpp:22-68
    rotate_to_partition_order /
    adjust_topology / allocate_partition allocator.hpp:30-57, allocator.cpp:23-99
    scale_threshold / initial_threshold  threshold.hpp:30-36, threshold.cpp:23-47
    gather_stats                         collectives.cpp:22-45 (accounting)
    Engine(cfg, opt).step() -> IterationRecord   engine.hpp:61-105, engine.cpp:274-350
    SyntheticStream                      workloads.hpp:89-99 (generated on device)
    topk_select / hard_threshold_select  baselines.hpp:25-34, baselines.cpp:26-46 (device)

std::invalid_argument maps to InvalidArgument (a ValueError) and
sparsim::EngineError to EngineError. Device pointers are plain integers
(e.g. torch.Tensor.data_ptr()); torch is used only to allocate them.
"""
import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _abi as A
from ._lib import (DeviceError, EngineError, InvalidArgument, Unsupported, check, lib)

__all__ = [
    "SparsifierConfig", "validate", "default_block_count", "PartitionTopology", "IndexRange",
    "build_topology", "partition_range", "rotate_to_partition_order", "AdjustStats",
    "adjust_topology", "Allocation", "allocate_partition", "scale_threshold",
    "initial_threshold_device", "GatherStats", "gather_stats", "EngineOptions",
    "IterationRecord", "Engine", "StreamSpec", "SyntheticStream", "InvalidArgument",
    "EngineError", "DeviceError", "Unsupported", "nccl_unique_id", "flush_l2", "format_csv",
    "summarize", "topk_select", "hard_threshold_select",
]


# ---------------------------------------------------------------- config ----
@dataclass
class SparsifierConfig:
    """config.hpp:28-45 (defaults identical)."""
    n: int = 4
    n_g: int = 1_000_000
    n_b: int = 256
    d: float = 0.001
    k: int = 0
    delta0: Optional[float] = None
    alpha: float = 1.25
    beta: float = 1.25
    gamma: float = 0.02
    blk_move: int = 1
    min_blk: int = 2
    eta: float = 1.0
    seed: int = 42
    max_density_cap: Optional[float] = None

    def to_c(self):
        c = A.exd_config()
        c.n, c.n_g, c.n_b, c.d, c.k = self.n, self.n_g, self.n_b, self.d, self.k
        if self.delta0 is not None:
            c.has_delta0, c.delta0 = 1, self.delta0
        c.alpha, c.beta, c.gamma = self.alpha, self.beta, self.gamma
        c.blk_move, c.min_blk, c.eta, c.seed = self.blk_move, self.min_blk, self.eta, self.seed
        if self.max_density_cap is not None:
            c.has_max_density_cap, c.max_density_cap = 1, self.max_density_cap
        return c


def validate(cfg: SparsifierConfig) -> SparsifierConfig:
    """config.cpp:28-51: returns a copy with k = llround(d * n_g)."""
    out = A.exd_config()
    check(lib().exd_validate(C.byref(cfg.to_c()), C.byref(out)))
    v = SparsifierConfig(**cfg.__dict__)
    v.k = out.k
    return v


def default_block_count(n: int) -> int:
    return lib().exd_default_block_count(n)


# -------------------------------------------------------------- topology ----
@dataclass
class PartitionTopology:
    """types.hpp:36-46"""
    sz_blk: int = 0
    blk_part: List[int] = field(default_factory=list)
    blk_pos: List[int] = field(default_factory=list)

    def partitions(self):
        return len(self.blk_part)

    def total_blocks(self):
        return sum(self.blk_part)

    def to_c(self):
        t = A.exd_topology()
        t.n, t.sz_blk = len(self.blk_part), self.sz_blk
        for i, (b, p) in enumerate(zip(self.blk_part, self.blk_pos)):
            t.blk_part[i], t.blk_pos[i] = b, p
        return t

    @staticmethod
    def from_c(t):
        return PartitionTopology(t.sz_blk, t.parts(), t.pos())


@dataclass
class IndexRange:
    st: int = 0
    end: int = 0

    def length(self):
        return self.end - self.st


def build_topology(n_g, n_b, n, min_blk, warning: Optional[list] = None) -> PartitionTopology:
    """partition.cpp:22-58. `warning`, when a list, receives the alignment warning."""
    t = A.exd_topology()
    buf = C.create_string_buffer(256)
    check(lib().exd_build_topology(n_g, n_b, n, min_blk, C.byref(t), buf, 256))
    if warning is not None and buf.value:
        warning.append(buf.value.decode())
    return PartitionTopology.from_c(t)


def partition_range(topo: PartitionTopology, p: int, n_g: int) -> IndexRange:
    st, end = C.c_int64(), C.c_int64()
    check(lib().exd_partition_range(C.byref(topo.to_c()), p, n_g, C.byref(st), C.byref(end)))
    return IndexRange(st.value, end.value)


def rotate_to_partition_order(k_rank, t, n):
    """allocator.cpp:23-38 (rank order in, partition order out)."""
    if len(k_rank) != n:
        raise InvalidArgument("partial-k length mismatch")
    src = (C.c_int64 * n)(*k_rank)
    out = (C.c_int64 * n)()
    check(lib().exd_rotate_to_partition_order(src, t, n, out))
    return list(out)


@dataclass
class AdjustStats:
    moves: int = 0
    skips: int = 0


def adjust_topology(topo: PartitionTopology, k_part: list, alpha, blk_move, min_blk, n_g):
    """allocator.cpp:40-90; updates `topo` and `k_part` in place."""
    n = topo.partitions()
    ct = topo.to_c()
    k = (C.c_int64 * n)(*k_part)
    mv, sk = C.c_int32(), C.c_int32()
    check(lib().exd_adjust_topology(C.byref(ct), k, alpha, blk_move, min_blk, n_g,
                                    C.byref(mv), C.byref(sk)))
    topo.blk_part[:], topo.blk_pos[:] = ct.parts(), ct.pos()
    k_part[:] = list(k)
    return AdjustStats(mv.value, sk.value)


@dataclass
class Allocation:
    partition: int
    range: IndexRange


def allocate_partition(topo: PartitionTopology, t, rank, n_g) -> Allocation:
    p, st, end = C.c_int32(), C.c_int64(), C.c_int64()
    check(lib().exd_allocate_partition(C.byref(topo.to_c()), t, rank, n_g, C.byref(p),
                                       C.byref(st), C.byref(end)))
    return Allocation(p.value, IndexRange(st.value, end.value))


def scale_threshold(k, k_prime, delta, beta, gamma) -> float:
    return lib().exd_scale_threshold(k, k_prime, delta, beta, gamma)


def initial_threshold_device(mags_ptr: int, m: int, d: float, dtype: str = "f32") -> float:
    """threshold.cpp:37-47 as a device radix select over |mags| (device pointer)."""
    out = C.c_double()
    check(lib().exd_initial_threshold_device(C.c_void_p(mags_ptr), m, _dtype_code(dtype), d,
                                             C.byref(out)))
    return out.value


def _acc_args(acc):
    """(device pointer, n_g, dtype code) of a contiguous CUDA fp32/fp64 tensor."""
    import torch
    if not (isinstance(acc, torch.Tensor) and acc.is_cuda and acc.dim() == 1
            and acc.is_contiguous() and acc.dtype in (torch.float32, torch.float64)):
        raise InvalidArgument("acc must be a contiguous 1-D CUDA float32/float64 tensor")
    code = A.EXD_F64 if acc.dtype == torch.float64 else A.EXD_F32
    return acc.data_ptr(), acc.numel(), code


def _stream_of(acc):
    import torch
    return C.c_void_p(torch.cuda.current_stream(acc.device).cuda_stream)


def topk_select(acc, k: int):
    """baselines.cpp:26-41: the k indices of largest |acc| (ties toward the
    lower index), ascending, as a device int32 tensor. Raises InvalidArgument
    ("topk_select: k out of range") unless 1 <= k <= acc.numel()."""
    import torch
    ptr, n_g, code = _acc_args(acc)
    out = torch.empty(max(k, 0), dtype=torch.int32, device=acc.device)
    with torch.cuda.device(acc.device):
        check(lib().exd_topk_select_device(C.c_void_p(ptr), n_g, code, k,
                                           C.c_void_p(out.data_ptr()), out.numel(),
                                           _stream_of(acc)))
    return out


def hard_threshold_select(acc, fixed_delta: float):
    """baselines.cpp:43-46: ascending {j : |acc[j]| >= fixed_delta} over the
    whole vector (compared in fp64), as a device int32 tensor."""
    import torch
    ptr, n_g, code = _acc_args(acc)
    out = torch.empty(n_g, dtype=torch.int32, device=acc.device)
    cnt = C.c_int64()
    with torch.cuda.device(acc.device):
        check(lib().exd_hard_threshold_select_device(C.c_void_p(ptr), n_g, code,
                                                     float(fixed_delta),
                                                     C.c_void_p(out.data_ptr()), out.numel(),
                                                     C.byref(cnt), _stream_of(acc)))
    return out[:cnt.value]


@dataclass
class GatherStats:
    k_prime: int
    m_t: int
    c_t: int
    f_t: float


def gather_stats(k_rank) -> GatherStats:
    n = len(k_rank)
    g = A.exd_gather_stats()
    check(lib().exd_gather_stats_of((C.c_int64 * n)(*k_rank), n, C.byref(g)))
    return GatherStats(g.k_prime, g.m_t, g.c_t, g.f_t)


# ---------------------------------------------------------------- engine ----
def _dtype_code(dtype):
    if dtype in ("f32", "float32", np.float32):
        return A.EXD_F32
    if dtype in ("f64", "float64", np.float64):
        return A.EXD_F64
    raise InvalidArgument("dtype out of range")


@dataclass
class EngineOptions:
    """engine.hpp:37-45 plus the device knobs (dtype, profile_kernels)."""
    sparsifier: str = "exdyna"
    static_partitions: bool = False
    fixed_delta: float = 0.0
    parallel_workers: bool = True
    verify_replication: bool = True
    verify_conservation: bool = False
    record_loss: bool = True
    dtype: str = "f32"
    profile_kernels: bool = False
    sync: str = "auto"          # one rank per GPU: "auto" | "nccl" | "p2p" | "p2p-pull"

    def to_c(self):
        o = A.exd_options()
        o.sparsifier = {"exdyna": 0, "topk": 1, "cltk": 2, "hardthreshold": 3}[self.sparsifier]
        o.static_partitions = int(self.static_partitions)
        o.fixed_delta = self.fixed_delta
        o.parallel_workers = int(self.parallel_workers)
        o.verify_replication = int(self.verify_replication)
        o.verify_conservation = int(self.verify_conservation)
        o.record_loss = int(self.record_loss)
        o.dtype = _dtype_code(self.dtype)
        o.profile_kernels = int(self.profile_kernels)
        o.sync_mode = {"auto": A.EXD_SYNC_AUTO, "nccl": A.EXD_SYNC_NCCL, "p2p": A.EXD_SYNC_P2P,
                       "p2p-pull": A.EXD_SYNC_P2P_PULL}[self.sync]
        return o


@dataclass
class IterationRecord:
    """types.hpp:84-103"""
    t: int = 0
    k_prime: int = 0
    density: float = 0.0
    eps: float = 0.0
    m_t: int = 0
    c_t: int = 0
    f_t: float = 1.0
    global_err: float = 0.0
    delta: float = 0.0
    loss: Optional[float] = None
    duplicates: int = 0
    union_count: int = 0
    k_rank: List[int] = field(default_factory=list)
    adjust_moves: int = 0
    adjust_skips: int = 0
    cap_hits: int = 0
    idle_workers: int = 0

    @staticmethod
    def from_c(r):
        return IterationRecord(**A.record_dict(r))


def _records_c(records):
    arr = (A.exd_record * max(1, len(records)))()
    for i, r in enumerate(records):
        c = arr[i]
        for f in A.RECORD_FIELDS:
            setattr(c, f, getattr(r, f))
        c.has_loss, c.loss = (1, r.loss) if r.loss is not None else (0, 0.0)
        c.n = len(r.k_rank)
        for j, k in enumerate(r.k_rank):
            c.k_rank[j] = k
    return arr


def format_csv(records) -> str:
    """runner.cpp:55-80 (same bytes as the reference's CSV ledger)."""
    arr = _records_c(records)
    n = C.c_size_t()
    check(lib().exd_format_csv(arr, len(records), None, 0, C.byref(n)))
    buf = C.create_string_buffer(n.value + 1)
    check(lib().exd_format_csv(arr, len(records), buf, n.value + 1, C.byref(n)))
    return buf.value.decode()


def summarize(records) -> dict:
    """runner.cpp:89-113 (RunStats)."""
    s = A.exd_run_stats()
    check(lib().exd_summarize(_records_c(records), len(records), C.byref(s)))
    out = {f: getattr(s, f) for f, _ in A.exd_run_stats._fields_ if not f.startswith("reserved")}
    out["final_loss"] = s.final_loss if s.has_final_loss else None
    del out["has_final_loss"]
    return out


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(A.NCCL_ID_BYTES)
    check(lib().exd_nccl_unique_id(buf))
    return buf.raw


def flush_l2(device=0, stream=0):
    check(lib().exd_flush_l2(device, C.c_void_p(stream)))


class Engine:
    """sparsim::Engine on the B200 (engine.hpp:61-105).

    Engine(cfg, opt)                    all cfg.n workers in this process on one GPU
    Engine.rank(cfg, opt, r, dev, id)   rank r of an n-process job, NCCL over NVLink
    """

    def __init__(self, cfg: SparsifierConfig, opt: Optional[EngineOptions] = None, device=0,
                 _handle=None):
        self.cfg = validate(cfg)
        self.opt = opt or EngineOptions()
        self.L = lib()
        self.esize = 8 if _dtype_code(self.opt.dtype) == A.EXD_F64 else 4
        self.np_dtype = np.float64 if self.esize == 8 else np.float32
        if _handle is None:
            h = C.c_void_p()
            devs = (C.c_int32 * 1)(device)
            check(self.L.exd_engine_create(C.byref(cfg.to_c()), C.byref(self.opt.to_c()), devs, 1,
                                           C.byref(h)))
            _handle = h
        self.h = _handle
        self.device = device
        self.local_workers = self.L.exd_engine_local_workers(self.h)
        self.first_rank = self.L.exd_engine_first_rank(self.h)

    @classmethod
    def rank(cls, cfg, opt, rank, device, nccl_id: bytes):
        opt = opt or EngineOptions()
        h = C.c_void_p()
        L = lib()
        check(L.exd_engine_create_rank(C.byref(cfg.to_c()), C.byref(opt.to_c()), rank, device,
                                       nccl_id, C.byref(h)))
        return cls(cfg, opt, device, _handle=h)

    def close(self):
        if getattr(self, "h", None):
            self.L.exd_engine_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # -- stepping ---------------------------------------------------------
    def _ptrs(self, grads):
        if len(grads) != self.local_workers:
            raise InvalidArgument("one gradient per local worker")
        ps = []
        for g in grads:
            if isinstance(g, int):  # a raw device pointer: the C ABI checks null / alignment
                ps.append(g)
                continue
            import torch
            want = torch.float64 if self.np_dtype == np.float64 else torch.float32
            if not (isinstance(g, torch.Tensor) and g.is_cuda):
                raise InvalidArgument("gradient must be a CUDA tensor or a device pointer")
            if g.dtype != want:
                raise InvalidArgument(f"gradient dtype {g.dtype} != engine dtype {want}")
            if g.numel() != self.cfg.n_g or not g.is_contiguous():
                raise InvalidArgument("engine: workload size != n_g")
            if g.device.index != self.device:
                raise InvalidArgument(f"gradient on {g.device}, engine on cuda:{self.device}")
            if g.data_ptr() % 16:
                raise InvalidArgument("gradient pointer must be 16-byte aligned")
            ps.append(g.data_ptr())
        return (C.c_void_p * len(ps))(*ps)

    def step(self, grads) -> IterationRecord:
        """Engine::step(): grads are device buffers (one per local worker)."""
        rec = A.exd_record()
        check(self.L.exd_engine_step(self.h, self._ptrs(grads), C.byref(rec)))
        return IterationRecord.from_c(rec)

    def step_async(self, grads):
        check(self.L.exd_engine_step_async(self.h, self._ptrs(grads)))

    def sync(self) -> IterationRecord:
        rec = A.exd_record()
        check(self.L.exd_engine_sync(self.h, C.byref(rec)))
        return IterationRecord.from_c(rec)

    def step_host(self, grads) -> IterationRecord:
        """Host-buffer step: grads are numpy arrays (pinned or pageable)."""
        arrs = [np.ascontiguousarray(g, dtype=self.np_dtype) for g in grads]
        ps = (C.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])
        rec = A.exd_record()
        check(self.L.exd_engine_step_host(self.h, ps, C.byref(rec)))
        return IterationRecord.from_c(rec)

    def run(self, iterations, source, device_bufs):
        """Engine::run (engine.cpp:352-357) over a device GradientSource: the
        generator and the steps are stream-ordered on the engine's stream, so
        steps are only enqueued here; the records are fetched in batches."""
        out = []
        first = self.iteration()
        for i in range(iterations):
            t = self.iteration()
            for w, buf in enumerate(device_bufs):
                source.gradient(t, self.first_rank + w, buf, self.opt.dtype, self.stream(w))
            self.step_async(device_bufs)
            if (i + 1) % 128 == 0 or i + 1 == iterations:
                out.extend(self.records(first + len(out), i + 1 - len(out)))
        return out

    def records(self, first, count):
        """IterationRecords of steps [first, first + count) (the device keeps
        the last EXD_RECORD_RING)."""
        if count <= 0:
            return []
        buf = (A.exd_record * count)()
        check(self.L.exd_engine_records(self.h, first, count, buf))
        return [IterationRecord.from_c(r) for r in buf]

    # -- state --------------------------------------------------------------
    def iteration(self):
        return self.L.exd_engine_iteration(self.h)

    def sync_mode(self):
        """'p2p' (push-reduce) / 'p2p-pull' / 'nccl' for a rank engine, 'in-process' otherwise."""
        return {-1: "in-process", A.EXD_SYNC_P2P: "p2p", A.EXD_SYNC_P2P_PULL: "p2p-pull",
                A.EXD_SYNC_NCCL: "nccl"}[
            self.L.exd_engine_sync_mode(self.h)]

    def stream(self, w=0):
        return self.L.exd_engine_stream(self.h, w) or 0

    def state(self, w=0):
        s = A.exd_worker_state()
        check(self.L.exd_engine_get_state(self.h, w, C.byref(s)))
        return s

    def delta(self, w=0):
        return self.state(w).delta

    def k_t(self, w=0):
        s = self.state(w)
        return list(s.k_t[: self.cfg.n])

    def topology(self, w=0) -> PartitionTopology:
        return PartitionTopology.from_c(self.state(w).topology)

    def _copy(self, w, which, dtype):
        n = C.c_int64()
        check(self.L.exd_engine_copy_out(self.h, w, which, None, 0, C.byref(n)))
        out = np.empty(n.value, dtype=dtype)
        if n.value:
            check(self.L.exd_engine_copy_out(self.h, w, which, C.c_void_p(out.ctypes.data),
                                             n.value, C.byref(n)))
        return out

    def x(self, w=0):
        return self._copy(w, A.EXD_VEC_X, self.np_dtype)

    def e(self, w=0):
        return self._copy(w, A.EXD_VEC_E, self.np_dtype)

    def idx_global(self, w=0):
        return self._copy(w, A.EXD_VEC_IDX_GLOBAL, np.int32)

    def selection(self, w=0):
        return self._copy(w, A.EXD_VEC_LOCAL_IDX, np.int32)

    def selected_values(self, w=0):
        return self._copy(w, A.EXD_VEC_LOCAL_VAL, self.np_dtype)

    def block_counts(self, w=0):
        return self._copy(w, A.EXD_VEC_BLOCK_COUNTS, np.int32)

    def reduced(self, w=0):
        return self._copy(w, A.EXD_VEC_SUM, self.np_dtype)

    def device_view(self, w, which):
        """Zero-copy torch view of x / e / idx_global / ... of worker w (device
        memory owned by the engine; valid until close())."""
        import torch
        code = {"x": A.EXD_VEC_X, "e": A.EXD_VEC_E, "idx_global": A.EXD_VEC_IDX_GLOBAL,
                "selection": A.EXD_VEC_LOCAL_IDX, "selected_values": A.EXD_VEC_LOCAL_VAL,
                "block_counts": A.EXD_VEC_BLOCK_COUNTS, "reduced": A.EXD_VEC_SUM}[which]
        ptr, n = C.c_void_p(), C.c_int64()
        check(self.L.exd_engine_device_vector(self.h, w, code, C.byref(ptr), C.byref(n)))
        int_vec = code in (A.EXD_VEC_IDX_GLOBAL, A.EXD_VEC_LOCAL_IDX, A.EXD_VEC_BLOCK_COUNTS)
        typestr = "<i4" if int_vec else ("<f8" if self.esize == 8 else "<f4")

        class _View:
            __cuda_array_interface__ = {"shape": (n.value,), "typestr": typestr,
                                        "data": (ptr.value or 0, False), "version": 3}
        return torch.as_tensor(_View(), device=f"cuda:{self.device}")

    def write(self, w, which, arr):
        """mutable_workers() (engine.hpp:72-74): overwrite x or e of worker w."""
        a = np.ascontiguousarray(arr, dtype=self.np_dtype)
        code = {"x": A.EXD_VEC_X, "e": A.EXD_VEC_E}[which]
        check(self.L.exd_engine_copy_in(self.h, w, code, C.c_void_p(a.ctypes.data), a.size))

    def kernel_stats(self):
        s = A.exd_kernel_stats()
        check(self.L.exd_engine_kernel_stats(self.h, C.byref(s)))
        return {"select_launches": s.select_launches, "select_ms": s.select_ms, "steps": s.steps,
                "kernel_launches": s.kernel_launches, "finish_launches": s.finish_launches,
                "finish_ms": s.finish_ms}

    def reset_kernel_stats(self):
        check(self.L.exd_engine_reset_kernel_stats(self.h))

    def set_profile(self, on: bool):
        check(self.L.exd_engine_set_profile(self.h, int(on)))


# ------------------------------------------------------------- workloads ----
@dataclass
class StreamSpec:
    """workloads.hpp:121-129"""
    n_g: int
    segments: list = None          # [(length, scale)]; None -> default 4-segment stream
    distribution: int = 0          # 0 Laplace, 1 LogNormal
    decay: float = 1.0
    decay_step: Optional[int] = None
    decay_step_factor: float = 0.1
    seed: int = 42

    def resolved_segments(self):
        if self.segments is not None:
            return list(self.segments)
        q = self.n_g // 4  # run_config.cpp:248-260
        if q > 0:
            return [(q, 1.0), (q, 0.5), (q, 0.25), (self.n_g - 3 * q, 0.125)]
        return [(self.n_g, 1.0)]

    def to_c(self):
        s = A.exd_stream_spec()
        segs = self.resolved_segments()
        s.n_g, s.nseg, s.distribution = self.n_g, len(segs), self.distribution
        for i, (ln, sc) in enumerate(segs):
            s.seg_length[i], s.seg_scale[i] = ln, sc
        s.decay, s.decay_step_factor, s.seed = self.decay, self.decay_step_factor, self.seed
        if self.decay_step is not None:
            s.has_decay_step, s.decay_step = 1, self.decay_step
        return s


class SyntheticStream:
    """SyntheticStream (workloads.hpp:166-176) generated on the device."""

    def __init__(self, spec: StreamSpec):
        self.spec = spec
        self._c = spec.to_c()

    def size(self):
        return self.spec.n_g

    def gradient(self, t, rank, out_ptr, dtype="f32", stream=0):
        ptr = out_ptr if isinstance(out_ptr, int) else out_ptr.data_ptr()
        check(lib().exd_synthetic_gradient(C.byref(self._c), t, rank, _dtype_code(dtype),
                                           C.c_void_p(ptr), C.c_void_p(stream)))
