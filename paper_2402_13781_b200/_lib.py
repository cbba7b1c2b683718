"""Loader for the in-tree libexdyna.so (the C ABI of include/exdyna.h).

The library is the product: there is no CPU fallback. If it is missing the
import of any engine entry point fails loudly.
"""
import ctypes as C
import os

from . import _abi as A

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("EXD_LIB") or os.path.join(HERE, "lib", "libexdyna.so")

_lib = None

P = C.c_void_p
PI64 = C.POINTER(C.c_int64)
PI32 = C.POINTER(C.c_int32)


class InvalidArgument(ValueError):
    """std::invalid_argument in the reference (config.cpp:29-49, engine.cpp:55-61)."""


class EngineError(RuntimeError):
    """sparsim::EngineError (engine.hpp:47-50): a violated engine invariant."""


class DeviceError(RuntimeError):
    """CUDA / NCCL failure inside the B200 path."""


class Unsupported(RuntimeError):
    """A reference option this build does not implement on the device path."""


def _sig(L, name, res, args):
    f = getattr(L, name)
    f.restype = res
    f.argtypes = args


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2402_13781_b200.build` "
            "(the B200 path has no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    _sig(L, "exd_last_error", C.c_char_p, [])
    _sig(L, "exd_version", C.c_int32, [])
    _sig(L, "exd_validate", C.c_int, [C.POINTER(A.exd_config), C.POINTER(A.exd_config)])
    _sig(L, "exd_default_block_count", C.c_int64, [C.c_int32])
    _sig(L, "exd_build_topology", C.c_int, [C.c_int64, C.c_int64, C.c_int32, C.c_int64,
                                            C.POINTER(A.exd_topology), C.c_char_p, C.c_size_t])
    _sig(L, "exd_partition_range", C.c_int, [C.POINTER(A.exd_topology), C.c_int32, C.c_int64,
                                             PI64, PI64])
    _sig(L, "exd_rotate_to_partition_order", C.c_int, [PI64, C.c_int64, C.c_int32, PI64])
    _sig(L, "exd_adjust_topology", C.c_int, [C.POINTER(A.exd_topology), PI64, C.c_double,
                                             C.c_int64, C.c_int64, C.c_int64, PI32, PI32])
    _sig(L, "exd_allocate_partition", C.c_int, [C.POINTER(A.exd_topology), C.c_int64, C.c_int32,
                                                C.c_int64, PI32, PI64, PI64])
    _sig(L, "exd_scale_threshold", C.c_double, [C.c_int64, C.c_int64, C.c_double, C.c_double,
                                                C.c_double])
    _sig(L, "exd_gather_stats_of", C.c_int, [PI64, C.c_int32, C.POINTER(A.exd_gather_stats)])
    _sig(L, "exd_initial_threshold_device", C.c_int, [P, C.c_int64, C.c_int32, C.c_double,
                                                      C.POINTER(C.c_double)])
    _sig(L, "exd_topk_select_device", C.c_int, [P, C.c_int64, C.c_int32, C.c_int64, P,
                                                C.c_int64, P])
    _sig(L, "exd_hard_threshold_select_device", C.c_int, [P, C.c_int64, C.c_int32, C.c_double,
                                                          P, C.c_int64, PI64, P])
    _sig(L, "exd_synthetic_gradient", C.c_int, [C.POINTER(A.exd_stream_spec), C.c_int64,
                                                C.c_int32, C.c_int32, P, P])
    _sig(L, "exd_engine_create", C.c_int, [C.POINTER(A.exd_config), C.POINTER(A.exd_options),
                                           PI32, C.c_int32, C.POINTER(P)])
    _sig(L, "exd_nccl_unique_id", C.c_int, [C.c_char_p])
    _sig(L, "exd_engine_create_rank", C.c_int, [C.POINTER(A.exd_config), C.POINTER(A.exd_options),
                                                C.c_int32, C.c_int32, C.c_char_p, C.POINTER(P)])
    _sig(L, "exd_engine_destroy", None, [P])
    _sig(L, "exd_engine_local_workers", C.c_int32, [P])
    _sig(L, "exd_engine_first_rank", C.c_int32, [P])
    _sig(L, "exd_engine_iteration", C.c_int64, [P])
    _sig(L, "exd_engine_sync_mode", C.c_int32, [P])
    _sig(L, "exd_engine_stream", P, [P, C.c_int32])
    _sig(L, "exd_engine_step", C.c_int, [P, C.POINTER(P), C.POINTER(A.exd_record)])
    _sig(L, "exd_engine_step_async", C.c_int, [P, C.POINTER(P)])
    _sig(L, "exd_engine_sync", C.c_int, [P, C.POINTER(A.exd_record)])
    _sig(L, "exd_engine_records", C.c_int, [P, C.c_int64, C.c_int64, C.POINTER(A.exd_record)])
    _sig(L, "exd_engine_step_host", C.c_int, [P, C.POINTER(P), C.POINTER(A.exd_record)])
    _sig(L, "exd_engine_get_state", C.c_int, [P, C.c_int32, C.POINTER(A.exd_worker_state)])
    _sig(L, "exd_engine_copy_out", C.c_int, [P, C.c_int32, C.c_int32, P, C.c_int64, PI64])
    _sig(L, "exd_engine_copy_in", C.c_int, [P, C.c_int32, C.c_int32, P, C.c_int64])
    _sig(L, "exd_engine_device_vector", C.c_int, [P, C.c_int32, C.c_int32, C.POINTER(P), PI64])
    _sig(L, "exd_engine_kernel_stats", C.c_int, [P, C.POINTER(A.exd_kernel_stats)])
    _sig(L, "exd_engine_reset_kernel_stats", C.c_int, [P])
    _sig(L, "exd_engine_set_profile", C.c_int, [P, C.c_int32])
    _sig(L, "exd_flush_l2", C.c_int, [C.c_int32, P])
    _sig(L, "exd_format_csv", C.c_int, [C.POINTER(A.exd_record), C.c_int64, C.c_char_p,
                                        C.c_size_t, C.POINTER(C.c_size_t)])
    _sig(L, "exd_summarize", C.c_int, [C.POINTER(A.exd_record), C.c_int64,
                                       C.POINTER(A.exd_run_stats)])
    _lib = L
    return L


def check(rc):
    """Map an EXD_* status to the reference's exception classes."""
    if rc == A.EXD_OK:
        return
    msg = lib().exd_last_error().decode()
    if rc == A.EXD_EINVAL:
        raise InvalidArgument(msg)
    if rc == A.EXD_EINVARIANT:
        raise EngineError(msg)
    if rc == A.EXD_EUNSUPPORTED:
        raise Unsupported(msg)
    raise DeviceError(f"[{rc}] {msg}")


EXPORTED = [
    "exd_last_error", "exd_version", "exd_validate", "exd_default_block_count",
    "exd_build_topology", "exd_partition_range", "exd_rotate_to_partition_order",
    "exd_adjust_topology", "exd_allocate_partition", "exd_scale_threshold",
    "exd_gather_stats_of", "exd_initial_threshold_device", "exd_synthetic_gradient",
    "exd_topk_select_device", "exd_hard_threshold_select_device",
    "exd_engine_create", "exd_nccl_unique_id", "exd_engine_create_rank", "exd_engine_destroy",
    "exd_engine_local_workers", "exd_engine_first_rank", "exd_engine_iteration",
    "exd_engine_sync_mode",
    "exd_engine_stream", "exd_engine_step", "exd_engine_step_async", "exd_engine_sync",
    "exd_engine_records",
    "exd_engine_step_host", "exd_engine_get_state", "exd_engine_copy_out", "exd_engine_copy_in",
    "exd_engine_device_vector",
    "exd_engine_kernel_stats", "exd_engine_reset_kernel_stats", "exd_engine_set_profile",
    "exd_flush_l2", "exd_format_csv", "exd_summarize",
]
