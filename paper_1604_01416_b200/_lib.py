"""ctypes binding of libdmath_b200.so (declarations mirror include/dmath_b200.h).

The library is the product: there is no Python or CPU fallback.  Importing
this module raises if the shared object is missing.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libdmath_b200.so")

i32, i64, u64, f64, vp = C.c_int32, C.c_int64, C.c_uint64, C.c_double, C.c_void_p


class Layout(C.Structure):
    _fields_ = [("kind", i32), ("worker_count", i32), ("global_rows", i64), ("global_cols", i64),
                ("block_rows", i64), ("block_cols", i64), ("custom", C.POINTER(i32)),
                ("custom_len", i64)]


class PoolStats(C.Structure):
    _fields_ = [("fresh_allocations", u64), ("reuses", u64), ("bytes_live", u64),
                ("bytes_pooled", u64), ("high_water", u64)]


class WorkerStats(C.Structure):
    _fields_ = [("peer_bytes_read", u64), ("local_bytes_read", u64), ("gemm_launches", u64),
                ("split_launches", u64), ("gemm_flops", f64), ("gemm_ms", f64)]


class Descriptor(C.Structure):
    _fields_ = [("matrix_id", u64), ("precision", i32), ("replicated", i32), ("version", u64),
                ("replica_version", u64), ("seed", u64), ("layout", Layout)]


class TransferRecord(C.Structure):
    _fields_ = [("seq", u64), ("src", i32), ("dst", i32), ("matrix_id", u64), ("row", i32), ("col", i32),
                ("bytes", u64), ("op", C.c_char * 32)]


class SessionConfig(C.Structure):
    _fields_ = [("worker_count", i32), ("mode", i32), ("rank", i32), ("coherence_checks", i32),
                ("root_seed", u64), ("devices", C.POINTER(i32)), ("nccl_id", vp), ("gemm_mode", i32)]


def _load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the B200 path has no fallback implementation)")
    lib = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
    P = C.POINTER
    sigs = {
        "dm_last_error": (C.c_char_p, []),
        "dm_last_error_missing": (C.c_int, [P(i32), C.c_int]),
        "dm_abi_version": (C.c_int, []),
        "dm_checkerboard_dims": (C.c_int, [C.c_int, P(C.c_int), P(C.c_int)]),
        "dm_layout_owner": (C.c_int, [P(Layout), C.c_int, C.c_int, P(C.c_int)]),
        "dm_layout_grid": (C.c_int, [P(Layout), P(C.c_int), P(C.c_int), P(C.c_int)]),
        "dm_block_extent": (C.c_int, [P(Layout), C.c_int, C.c_int, P(i64), P(i64)]),
        "dm_layout_to_string": (C.c_int, [P(Layout), C.c_char_p, C.c_int]),
        "dm_pool_size_class": (u64, [u64]),
        "dm_plan_general_gemm": (C.c_int, [P(Layout), C.c_int, P(Layout), C.c_int, P(Layout),
                                           C.c_int, P(i64), P(i64)]),
        "dm_session_create": (C.c_int, [P(SessionConfig), P(vp)]),
        "dm_session_destroy": (C.c_int, [vp]),
        "dm_session_shutdown": (C.c_int, [vp]),
        "dm_nccl_unique_id": (C.c_int, [vp]),
        "dm_create_matrix": (C.c_int, [vp, P(Layout), C.c_int, C.c_int, vp, P(u64)]),
        "dm_destroy_matrix": (C.c_int, [vp, u64]),
        "dm_scatter": (C.c_int, [vp, u64, vp, i64, i64]),
        "dm_gather": (C.c_int, [vp, u64, vp, i64, i64, C.c_int]),
        "dm_update_block": (C.c_int, [vp, u64, C.c_int, C.c_int, vp, i64, i64]),
        "dm_replicate": (C.c_int, [vp, u64, C.c_int]),
        "dm_replica_read": (C.c_int, [vp, u64, C.c_int, vp, i64, i64]),
        "dm_reshape": (C.c_int, [vp, u64, P(Layout), C.c_int, P(u64)]),
        "dm_add_row_col_sum": (C.c_int, [vp, u64, C.c_int, C.c_int, P(u64)]),
        "dm_checkpoint": (C.c_int, [vp, C.c_char_p]),
        "dm_restore": (C.c_int, [C.c_char_p, P(SessionConfig), P(vp)]),
        "dm_general_gemm": (C.c_int, [vp, f64, u64, u64, f64, u64, C.c_int, C.c_int]),
        "dm_cyclic_gemm": (C.c_int, [vp, f64, u64, u64, f64, u64, C.c_int, C.c_int, C.c_int]),
        "dm_broadcast_gemm_reference": (C.c_int, [vp, f64, u64, u64, f64, u64, C.c_int, C.c_int]),
        "dm_cached_backward_gemm": (C.c_int, [vp, u64, u64, u64]),
        "dm_worker_count": (C.c_int, [vp, P(C.c_int)]),
        "dm_local_workers": (C.c_int, [vp, P(i32), C.c_int]),
        "dm_descriptor_get": (C.c_int, [vp, u64, P(Descriptor)]),
        "dm_pool_stats_get": (C.c_int, [vp, C.c_int, P(PoolStats)]),
        "dm_pool_trim": (C.c_int, [vp, C.c_int, P(u64)]),
        "dm_worker_stats_get": (C.c_int, [vp, C.c_int, P(WorkerStats)]),
        "dm_worker_stats_reset": (C.c_int, [vp]),
        "dm_set_gemm_timing": (C.c_int, [vp, C.c_int]),
        "dm_worker_seed": (C.c_int, [vp, C.c_int, P(u64)]),
        "dm_seed_workers": (C.c_int, [vp, u64, P(u64), C.c_int]),
        "dm_root_seed": (C.c_int, [vp, P(u64)]),
        "dm_transfer_log": (C.c_int, [vp, P(TransferRecord), C.c_int]),
        "dm_descriptor_digest": (C.c_int, [vp, P(u64), P(u64), C.c_int]),
        "dm_block_device_ptr": (C.c_int, [vp, u64, C.c_int, C.c_int, P(vp), P(C.c_int)]),
        "dm_barrier": (C.c_int, [vp]),
        "dm_set_async": (C.c_int, [vp, C.c_int]),
        "dm_marker_record": (C.c_int, [vp, C.c_int, C.c_int]),
        "dm_marker_elapsed": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_float)]),
        "dm_local_gemm_f32": (C.c_int, [f64, vp, i64, C.c_int, vp, i64, C.c_int, f64, vp, i64,
                                        i64, i64, i64, vp]),
        "dm_local_gemm_f32_ex": (C.c_int, [f64, vp, i64, C.c_int, vp, i64, C.c_int, f64, vp, i64,
                                           i64, i64, i64, C.c_int, C.c_int, vp]),
        "dm_local_gemm_f32_workspace_size": (C.c_int, [i64, i64, i64, C.c_int, C.c_int, P(C.c_size_t)]),
        "dm_local_gemm_f32_ws": (C.c_int, [f64, vp, i64, C.c_int, vp, i64, C.c_int, f64, vp, i64,
                                           i64, i64, i64, C.c_int, C.c_int, vp, C.c_size_t, vp]),
        "dm_session_gemm_mode": (C.c_int, [vp, P(C.c_int)]),
        "dm_split_mode_for": (C.c_int, [C.c_int, i64, C.c_double, P(C.c_int)]),
        "dm_presplit_panels": (C.c_int, [i64, i64, i64, i64, P(C.c_int64), C.c_int, P(C.c_int)]),
        "dm_fill_seeded_f32": (C.c_int, [vp, i64, u64, C.c_int, C.c_int, vp]),
    }
    for name, (res, args) in sigs.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()

# names of every symbol include/dmath_b200.h declares (checked by the CPU tests)
EXPORTED = [
    "dm_last_error", "dm_last_error_missing", "dm_abi_version", "dm_checkerboard_dims",
    "dm_layout_owner", "dm_layout_grid", "dm_block_extent", "dm_layout_to_string",
    "dm_pool_size_class", "dm_plan_general_gemm", "dm_session_create", "dm_session_destroy",
    "dm_session_shutdown", "dm_nccl_unique_id", "dm_create_matrix", "dm_destroy_matrix",
    "dm_scatter", "dm_gather", "dm_update_block", "dm_replicate", "dm_replica_read", "dm_reshape",
    "dm_add_row_col_sum", "dm_checkpoint", "dm_restore", "dm_general_gemm", "dm_cyclic_gemm", "dm_broadcast_gemm_reference",
    "dm_cached_backward_gemm", "dm_worker_count", "dm_local_workers", "dm_descriptor_get",
    "dm_pool_stats_get", "dm_pool_trim", "dm_worker_stats_get", "dm_worker_stats_reset",
    "dm_set_gemm_timing", "dm_worker_seed", "dm_seed_workers", "dm_root_seed", "dm_transfer_log", "dm_descriptor_digest", "dm_block_device_ptr",
    "dm_barrier", "dm_set_async", "dm_marker_record", "dm_marker_elapsed", "dm_local_gemm_f32", "dm_local_gemm_f32_ex", "dm_fill_seeded_f32",
    "dm_local_gemm_f32_workspace_size", "dm_local_gemm_f32_ws", "dm_session_gemm_mode",
    "dm_split_mode_for", "dm_presplit_panels",
]
