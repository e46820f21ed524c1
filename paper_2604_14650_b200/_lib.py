"""ctypes binding of the in-tree C ABI library ``lib/liblpm6cu.so`` (include/lpm6cu.h).

The library is the product: host C++ FIB build + sm_100a lookup kernels. There is
no fallback — if the library is missing, importing the lookup API raises.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
LIB_PATH = PKG_DIR / "lib" / "liblpm6cu.so"

# lpm6::Errc (types.hpp:27-40) + B200 additions; status = index + 1.
ERRC_NAMES = [
    "MalformedAddress", "UnsupportedPrefixLength", "MissingNextHop", "ReservedNextHop",
    "DuplicatePrefix", "UnknownPrefix", "SentinelCollision", "ExhaustedPrefixSpace",
    "InvalidArgument", "BadTraceFile", "BadSnapshotFile", "Io", "CudaError", "NcclError",
]

MAX_LEVELS = 9


class Lpm6Error(RuntimeError):
    """Mirror of lpm6::Error (types.hpp:42-49): carries the Errc name in ``code``."""

    def __init__(self, status: int, message: str):
        self.status = status
        self.code = ERRC_NAMES[status - 1] if 1 <= status <= len(ERRC_NAMES) else f"status{status}"
        super().__init__(f"{self.code}: {message}")


class Prefix_t(C.Structure):
    _fields_ = [("value_lo", C.c_uint64), ("value_hi", C.c_uint64), ("length", C.c_int32),
                ("next_hop", C.c_uint32), ("reserved", C.c_uint64)]


class Geometry_t(C.Structure):
    _fields_ = [("k", C.c_uint32), ("b", C.c_uint32), ("depth", C.c_uint32), ("value_bytes", C.c_uint32),
                ("leaf_keys", C.c_uint32), ("image_levels", C.c_uint32),
                ("num_keys", C.c_uint64), ("leaf_nodes", C.c_uint64), ("total_words", C.c_uint64),
                ("image_start", C.c_uint64),
                ("level_nodes", C.c_uint64 * MAX_LEVELS), ("level_start", C.c_uint64 * MAX_LEVELS),
                ("default_next_hop", C.c_uint32), ("leaf_image", C.c_uint32), ("leaf_words", C.c_uint32),
                ("reserved", C.c_uint32)]


class BuildOpts_t(C.Structure):
    _fields_ = [("merge_adjacent", C.c_uint32), ("value_bytes", C.c_uint32), ("leaf_format", C.c_uint32),
                ("reserved", C.c_uint32)]


class KernelConfig_t(C.Structure):
    _fields_ = [("lanes_per_query", C.c_uint32), ("smem_levels", C.c_uint32), ("ctas_per_sm", C.c_uint32),
                ("threads_per_cta", C.c_uint32), ("queries_per_lane", C.c_uint32), ("min_ctas_per_sm", C.c_uint32),
                ("line_path", C.c_uint32), ("plane_levels", C.c_uint32)]


class WorkloadInfo_t(C.Structure):
    _fields_ = [("id", C.c_int32), ("fib_kind", C.c_int32), ("n_queries", C.c_uint64), ("chunk", C.c_uint64),
                ("value_bytes", C.c_uint32), ("reserved", C.c_uint32), ("name", C.c_char * 8)]


class UpdateOp_t(C.Structure):
    _fields_ = [("kind", C.c_uint32), ("reserved0", C.c_uint32), ("reserved1", C.c_uint64), ("prefix", Prefix_t)]


class StoreStats_t(C.Structure):
    _fields_ = [("epoch", C.c_uint64), ("pending_ops", C.c_uint64), ("active_rules", C.c_uint64),
                ("retired", C.c_uint64), ("reclaimed", C.c_uint64), ("commits", C.c_uint64),
                ("last_build_ms", C.c_double), ("last_publish_us", C.c_double), ("fences", C.c_uint64)]


class Footprint_t(C.Structure):
    _fields_ = [("leaf_bytes", C.c_uint64), ("internal_bytes", C.c_uint64), ("value_bytes", C.c_uint64),
                ("image_bytes", C.c_uint64), ("total_bytes", C.c_uint64), ("bytes_per_interval", C.c_double),
                ("total_bytes_value8", C.c_uint64), ("bytes_per_interval_value8", C.c_double)]


P = C.c_void_p
U64 = C.c_uint64
U32 = C.c_uint32
I32 = C.c_int

# name -> (restype, argtypes); every symbol include/lpm6cu.h declares.
SIGNATURES = {
    "lpm6cu_last_error": (C.c_char_p, []),
    "lpm6cu_status_name": (C.c_char_p, [I32]),
    "lpm6cu_version": (C.c_char_p, []),
    "lpm6_build_intervals": (I32, [P, U64, U32, I32, P, P, U64, C.POINTER(U64)]),
    "lpm6_plan_layout": (I32, [U64, U32, C.POINTER(Geometry_t)]),
    "lpm6_build_tree": (I32, [P, P, U64, U32, U32, C.POINTER(Geometry_t), P, P]),
    "lpm6_plan_layout_ex": (I32, [U64, U32, U32, C.POINTER(Geometry_t)]),
    "lpm6_build_tree_ex": (I32, [P, P, U64, U32, U32, U32, C.POINTER(Geometry_t), P, P]),
    "lpm6_parse_prefix": (I32, [C.c_char_p, C.POINTER(Prefix_t), C.POINTER(I32)]),
    "lpm6cu_fib_build": (I32, [I32, P, U64, U32, C.POINTER(BuildOpts_t), C.POINTER(P)]),
    "lpm6cu_fib_build_device": (I32, [I32, P, U64, U32, C.POINTER(BuildOpts_t), P, C.POINTER(P)]),
    "lpm6cu_build_intervals_device": (I32, [I32, P, U64, U32, I32, P, P, U64, C.POINTER(U64)]),
    "lpm6cu_fib_create": (I32, [I32, C.POINTER(Geometry_t), P, C.POINTER(P)]),
    "lpm6cu_fib_wrap_device": (I32, [I32, C.POINTER(Geometry_t), P, C.POINTER(P)]),
    "lpm6cu_fib_adopt_device": (I32, [I32, C.POINTER(Geometry_t), P, C.POINTER(P)]),
    "lpm6cu_fib_replicate": (I32, [P, C.POINTER(I32), I32, P]),
    "lpm6cu_fib_geometry": (I32, [P, C.POINTER(Geometry_t)]),
    "lpm6cu_fib_device_lines": (I32, [P, C.POINTER(P)]),
    "lpm6cu_fib_copy_lines": (I32, [P, P, U64]),
    "lpm6cu_fib_set_kernel_config": (I32, [P, C.POINTER(KernelConfig_t)]),
    "lpm6cu_fib_kernel_config": (I32, [P, C.POINTER(KernelConfig_t)]),
    "lpm6cu_fib_tune_line_path": (I32, [P, P, U64, P, P, U32, C.POINTER(U32)]),
    "lpm6cu_fib_destroy": (None, [P]),
    "lpm6cu_fib_set_checked": (I32, [P, I32]),
    "lpm6cu_fib_violations": (I32, [P, C.POINTER(U32), I32]),
    "lpm6cu_fib_node_visits": (I32, [P, C.POINTER(U64), I32]),
    "lpm6cu_lookup_batch": (I32, [P, P, U64, P, P]),
    "lpm6cu_lookup_batch_device": (I32, [P, P, U64, P, P]),
    "lpm6_workload_info_get": (I32, [I32, C.POINTER(WorkloadInfo_t)]),
    "lpm6_workload_fib": (I32, [I32, P, U64, C.POINTER(U64), C.POINTER(U32)]),
    "lpm6_workload_queries_host": (I32, [I32, P, U64, U64, U64, P, I32]),
    "lpm6cu_querygen_create": (I32, [I32, I32, P, U64, C.POINTER(P)]),
    "lpm6cu_querygen_run": (I32, [P, U64, U64, P, P]),
    "lpm6cu_querygen_destroy": (None, [P]),
    "lpm6cu_probe_l2_gather": (I32, [I32, U64, U32, C.POINTER(C.c_double)]),
    "lpm6cu_probe_smem": (I32, [I32, C.POINTER(C.c_double)]),
    "lpm6cu_lookup_keys": (I32, [P, P, U64, P, P]),
    "lpm6cu_lookup_packets": (I32, [P, P, U64, U64, U32, P, P]),
    "lpm6cu_search_batch": (I32, [P, P, U64, P, P, P]),
    "lpm6cu_fib_build_from_intervals": (I32, [I32, P, P, U64, U32, C.POINTER(BuildOpts_t), P, C.POINTER(P)]),
    "lpm6_snapshot_encode": (I32, [P, P, U64, U32, P, U64, C.POINTER(U64)]),
    "lpm6_snapshot_save": (I32, [P, P, U64, U32, C.c_char_p]),
    "lpm6_snapshot_decode": (I32, [P, U64, P, P, U64, C.POINTER(U64), C.POINTER(U32)]),
    "lpm6cu_fib_load_snapshot": (I32, [I32, C.c_char_p, U32, C.POINTER(BuildOpts_t), P, C.POINTER(P)]),
    "lpm6_trace_save": (I32, [P, U64, C.c_char_p]),
    "lpm6_memory_footprint": (I32, [C.POINTER(Geometry_t), C.POINTER(Footprint_t)]),
    "lpm6_ref_memory_footprint": (I32, [U64, U32, C.POINTER(Footprint_t)]),
    "lpm6_trace_count": (I32, [P, U64, C.POINTER(U64)]),
    "lpm6cu_trace_load": (I32, [I32, C.c_char_p, P, U64, C.POINTER(U64), P]),
    "lpm6_parse_update": (I32, [C.c_char_p, C.POINTER(UpdateOp_t)]),
    "lpm6_apply_updates": (I32, [P, U64, P, U64, P, U64, C.POINTER(U64), C.POINTER(U64), P]),
    "lpm6cu_store_create": (I32, [I32, P, U64, U32, C.POINTER(BuildOpts_t), C.POINTER(P)]),
    "lpm6cu_store_destroy": (I32, [P]),
    "lpm6cu_store_stage": (I32, [P, P, U64, C.POINTER(U64), P]),
    "lpm6cu_store_commit": (I32, [P, C.POINTER(U64)]),
    "lpm6cu_store_acquire": (I32, [P, C.POINTER(P)]),
    "lpm6cu_store_release": (I32, [P, P]),
    "lpm6cu_snapshot_info": (I32, [P, C.POINTER(U64), C.POINTER(P), C.POINTER(U64)]),
    "lpm6cu_snapshot_rules": (I32, [P, P, U64]),
    "lpm6cu_store_lookup_batch": (I32, [P, P, U64, P, P, C.POINTER(U64)]),
    "lpm6cu_store_reclaim": (I32, [P]),
    "lpm6cu_store_stats_get": (I32, [P, C.POINTER(StoreStats_t)]),
}

_lib = None


def lib() -> C.CDLL:
    """Load the library once; raise loudly when it has not been built."""
    global _lib
    if _lib is None:
        path = Path(os.environ.get("LPM6CU_LIB", LIB_PATH))
        if not path.exists():
            raise ImportError(f"{path} is missing: run __graft_entry__.build() (make -C "
                              f"paper_2604_14650_b200/csrc); there is no CPU fallback")
        handle = C.CDLL(str(path))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def check(status: int) -> None:
    if status != 0:
        msg = lib().lpm6cu_last_error().decode(errors="replace")
        raise Lpm6Error(status, msg)
