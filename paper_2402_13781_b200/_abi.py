"""ctypes mirror of include/exdyna.h (the C ABI of the B200 ExDyna path).

Struct layouts must match the header field for field; tests/test_capi.py
checks the sizes against the library's own sizeof() exports.
"""
import ctypes as C

MAX_WORKERS = 64
MAX_SEGMENTS = 64
NCCL_ID_BYTES = 128

EXD_OK, EXD_EINVAL, EXD_EINVARIANT, EXD_ECUDA, EXD_ENCCL, EXD_ENOMEM, EXD_EUNSUPPORTED = range(7)
EXD_F32, EXD_F64 = 0, 1
EXD_SYNC_AUTO, EXD_SYNC_NCCL, EXD_SYNC_P2P, EXD_SYNC_P2P_PULL = 0, 1, 2, 3
EXD_SPARSIFIER_EXDYNA, EXD_SPARSIFIER_TOPK, EXD_SPARSIFIER_CLTK, EXD_SPARSIFIER_HARD_THRESHOLD = range(4)
(EXD_VEC_X, EXD_VEC_E, EXD_VEC_IDX_GLOBAL, EXD_VEC_LOCAL_IDX, EXD_VEC_LOCAL_VAL,
 EXD_VEC_BLOCK_COUNTS, EXD_VEC_SUM) = range(7)

i32, i64, u64, f64 = C.c_int32, C.c_int64, C.c_uint64, C.c_double


class exd_config(C.Structure):
    _fields_ = [
        ("n", i32), ("has_delta0", i32), ("n_g", i64), ("n_b", i64), ("d", f64),
        ("k", i64), ("delta0", f64), ("alpha", f64), ("beta", f64), ("gamma", f64),
        ("blk_move", i64), ("min_blk", i64), ("eta", f64), ("seed", u64),
        ("has_max_density_cap", i32), ("reserved0", i32), ("max_density_cap", f64),
    ]


class exd_options(C.Structure):
    _fields_ = [
        ("sparsifier", i32), ("static_partitions", i32), ("fixed_delta", f64),
        ("parallel_workers", i32), ("verify_replication", i32),
        ("verify_conservation", i32), ("record_loss", i32), ("dtype", i32),
        ("profile_kernels", i32), ("sync_mode", i32),
    ]


class exd_topology(C.Structure):
    _fields_ = [
        ("n", i32), ("reserved0", i32), ("sz_blk", i64),
        ("blk_part", i64 * MAX_WORKERS), ("blk_pos", i64 * MAX_WORKERS),
    ]

    def parts(self):
        return list(self.blk_part[: self.n])

    def pos(self):
        return list(self.blk_pos[: self.n])


class exd_record(C.Structure):
    _fields_ = [
        ("t", i64), ("k_prime", i64), ("density", f64), ("eps", f64),
        ("m_t", i64), ("c_t", i64), ("f_t", f64), ("global_err", f64),
        ("delta", f64), ("has_loss", i32), ("reserved0", i32), ("loss", f64),
        ("duplicates", i64), ("union_count", i64), ("n", i32),
        ("adjust_moves", i32), ("adjust_skips", i32), ("cap_hits", i32),
        ("idle_workers", i32), ("reserved1", i32), ("k_rank", i64 * MAX_WORKERS),
    ]

    def krank(self):
        return list(self.k_rank[: self.n])


class exd_gather_stats(C.Structure):
    _fields_ = [("k_prime", i64), ("m_t", i64), ("c_t", i64), ("f_t", f64)]


class exd_worker_state(C.Structure):
    _fields_ = [
        ("t", i64), ("rank", i32), ("partition", i32), ("delta", f64),
        ("st", i64), ("end", i64), ("k_t", i64 * MAX_WORKERS), ("topology", exd_topology),
    ]


class exd_stream_spec(C.Structure):
    _fields_ = [
        ("n_g", i64), ("nseg", i32), ("distribution", i32),
        ("seg_length", i64 * MAX_SEGMENTS), ("seg_scale", f64 * MAX_SEGMENTS),
        ("decay", f64), ("has_decay_step", i32), ("reserved0", i32),
        ("decay_step", i64), ("decay_step_factor", f64), ("seed", u64),
    ]


class exd_kernel_stats(C.Structure):
    _fields_ = [("select_launches", i64), ("select_ms", f64), ("steps", i64),
                ("kernel_launches", i64), ("finish_launches", i64), ("finish_ms", f64)]


class exd_run_stats(C.Structure):
    _fields_ = [("iterations", i64), ("mean_density", f64), ("mean_f", f64), ("mean_eps", f64),
                ("duplicates", i64), ("adjust_moves", i64), ("adjust_skips", i64),
                ("cap_hits", i64), ("mean_idle_workers", f64), ("final_delta", f64),
                ("final_global_err", f64), ("has_final_loss", i32), ("reserved0", i32),
                ("final_loss", f64)]


RECORD_FIELDS = ("t", "k_prime", "density", "eps", "m_t", "c_t", "f_t", "global_err",
                 "delta", "duplicates", "union_count", "adjust_moves", "adjust_skips",
                 "cap_hits", "idle_workers")


def record_dict(rec):
    out = {f: getattr(rec, f) for f in RECORD_FIELDS}
    out["k_rank"] = rec.krank()
    out["loss"] = rec.loss if rec.has_loss else None
    return out
