"""ctypes binding of libopflow_b200.so (the C-ABI in include/opflow_b200.h).

The shared object is built in-tree (paper_2605_21603_b200/build.py); loading
fails loudly if it is missing — there is no Python or CPU fallback for the
device path.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_PKG = Path(__file__).resolve().parent
# OPF_LIB overrides the library (A/B timing of a variant build, tools/build_ab.py)
LIB_PATH = Path(os.environ["OPF_LIB"]) if os.environ.get("OPF_LIB") else _PKG / "libopflow_b200.so"

ERRC = [
    "CycleDetected", "UnknownTensor", "ShapeMismatch", "DuplicateId", "MissingBinding",
    "SizeMismatch", "SplitReplicated", "OverlappingRules", "NonContiguousRegion", "PlanInvariant",
    "UnknownSubgraph", "UseAfterFree", "Unmaterialized", "DoubleProduce", "AlreadySplit",
    "InvalidUbatch", "NotReady", "DuplicateHandle", "SignatureMismatch", "MergeAcrossSplits",
    "IncompleteSchedule", "SchedulerError", "EngineStopped", "MissingLabels", "MissingPattern",
    "ConfigError",
]


class opf_view(C.Structure):
    _fields_ = [("base", C.c_void_p), ("elem_offset", C.c_int64), ("dtype", C.c_int32),
                ("rank", C.c_int32), ("shape", C.c_int64 * 4), ("batched", C.c_int32),
                ("_pad", C.c_int32)]


class opf_op_ctx(C.Structure):
    _fields_ = [("op_name", C.c_char_p), ("kind", C.c_int32), ("custom_name", C.c_char_p),
                ("world_size", C.c_int64), ("seed", C.c_uint64), ("n_params", C.c_int32),
                ("param_names", C.POINTER(C.c_char_p)), ("param_values", C.POINTER(C.c_double)),
                ("max_ctas", C.c_int32), ("_pad", C.c_int32), ("comm", C.c_void_p),
                ("aux", C.c_void_p), ("workspace", C.c_void_p), ("workspace_bytes", C.c_size_t)]


class opf_handle(C.Structure):
    _fields_ = [("subgraph", C.c_int32), ("ubatch", C.c_int32), ("topo_index", C.c_int32)]


KERNEL_FN = C.CFUNCTYPE(C.c_int32, C.POINTER(opf_op_ctx), C.POINTER(opf_view), C.c_int32,
                        C.POINTER(opf_view), C.c_int32, C.c_int64, C.c_void_p)
SCHEDULE_FN = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.c_void_p)

_SIGS = {
    "opf_last_error": (C.c_char_p, []),
    "opf_errc_name": (C.c_char_p, [C.c_int32]),
    "opf_version": (C.c_char_p, []),
    "opf_free_string": (None, [C.c_void_p]),
    "opf_graph_build": (C.c_int32, [C.c_char_p, C.POINTER(C.c_void_p)]),
    "opf_graph_free": (None, [C.c_void_p]),
    "opf_graph_dump": (C.c_int32, [C.c_void_p, C.POINTER(C.c_void_p)]),
    "opf_graph_tensor_id": (C.c_int32, [C.c_void_p, C.c_char_p, C.POINTER(C.c_int32)]),
    "opf_partition": (C.c_int32, [C.c_void_p, C.c_char_p, C.POINTER(C.c_void_p)]),
    "opf_plan_from_json": (C.c_int32, [C.c_void_p, C.c_char_p, C.POINTER(C.c_void_p)]),
    "opf_validate_plan": (C.c_int32, [C.c_void_p, C.c_void_p]),
    "opf_plan_dump": (C.c_int32, [C.c_void_p, C.POINTER(C.c_void_p)]),
    "opf_plan_free": (None, [C.c_void_p]),
    "opf_builder_json": (C.c_int32, [C.c_char_p, C.c_char_p, C.POINTER(C.c_void_p)]),
    "opf_alltoall_permutation": (C.c_int32, [C.c_uint64, C.c_uint32, C.POINTER(C.c_uint32)]),
    "opf_register_op": (C.c_int32, [C.c_char_p, KERNEL_FN, C.c_int32, C.c_int32, C.c_int32]),
    "opf_has_op": (C.c_int32, [C.c_char_p, C.POINTER(C.c_int32)]),
    "opf_launch": (C.c_int32, [C.c_char_p, C.POINTER(opf_view), C.c_int32, C.POINTER(opf_view),
                               C.c_int32, C.c_int64, C.c_void_p]),
    "opf_gemm_splits": (C.c_int32, [C.c_int64, C.c_int64, C.c_int64, C.c_int32]),
    "opf_kv_create": (C.c_int32, [C.c_int32, C.c_int64, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                  C.c_int32, C.POINTER(C.c_void_p)]),
    "opf_kv_free": (None, [C.c_void_p]),
    "opf_kv_cache_ptr": (C.c_int32, [C.c_void_p, C.c_int32, C.c_int32, C.POINTER(C.c_void_p)]),
    "opf_kv_append": (C.c_int32, [C.c_void_p, C.POINTER(C.c_int64), C.POINTER(C.c_int32), C.c_int32,
                                  C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "opf_kv_release": (C.c_int32, [C.c_void_p, C.c_int64]),
    "opf_kv_block_table": (C.c_int32, [C.c_void_p, C.POINTER(C.c_int64), C.c_int32, C.c_int64,
                                       C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "opf_kv_stats": (C.c_int32, [C.c_void_p, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "opf_view_rows": (C.c_int32, [C.POINTER(opf_view), C.c_int64, C.c_int64, C.POINTER(opf_view)]),
    "opf_comm_unique_id": (C.c_int32, [C.POINTER(C.c_uint8)]),
    "opf_comm_init": (C.c_int32, [C.POINTER(C.c_uint8), C.c_int32, C.c_int32, C.c_int32,
                                  C.POINTER(C.c_void_p)]),
    "opf_comm_free": (None, [C.c_void_p]),
    "opf_comm_window_set_epochs": (C.c_int32, [C.c_void_p, C.c_uint32]),
    "opf_comm_init_peer": (C.c_int32, [C.c_int32, C.c_int32, C.c_int32, C.POINTER(C.c_void_p)]),
    "opf_session_check": (C.c_int32, [C.c_void_p]),
    "opf_comm_window_alloc": (C.c_int32, [C.c_void_p, C.c_size_t, C.POINTER(C.c_uint8)]),
    "opf_comm_window_open": (C.c_int32, [C.c_void_p, C.POINTER(C.c_uint8)]),
    "opf_comm_create_virtual": (C.c_int32, [C.c_int32, C.c_int32, C.c_size_t, C.POINTER(C.c_void_p)]),
    "opf_comm_window_error": (C.c_int32, [C.c_void_p, C.POINTER(C.c_uint32)]),
    "opf_comm_push_calls": (C.c_int32, [C.c_void_p, C.POINTER(C.c_uint32)]),
    "opf_launch_comm": (C.c_int32, [C.c_char_p, C.POINTER(opf_view), C.c_int32, C.POINTER(opf_view),
                                    C.c_int32, C.c_int64, C.c_void_p, C.c_int32, C.c_void_p]),
    "opf_session_create": (C.c_int32, [C.c_void_p, C.c_void_p, C.c_char_p, C.c_void_p,
                                       C.POINTER(C.c_void_p)]),
    "opf_session_free": (None, [C.c_void_p]),
    "opf_session_bind": (C.c_int32, [C.c_void_p, C.c_char_p, C.POINTER(opf_view)]),
    "opf_session_run": (C.c_int32, [C.c_void_p, C.c_char_p, C.c_void_p]),
    "opf_session_prepare": (C.c_int32, [C.c_void_p, C.c_char_p, C.c_void_p]),
    "opf_session_arena_export": (C.c_int32, [C.c_void_p, C.c_int64, C.c_void_p]),
    "opf_session_arena_open": (C.c_int32, [C.c_void_p, C.c_void_p]),
    "opf_session_arena_link_local": (C.c_int32, [C.c_void_p, C.c_int32, C.c_int64]),
    "opf_session_run_custom": (C.c_int32, [C.c_void_p, C.c_char_p, SCHEDULE_FN, C.c_void_p,
                                           C.c_void_p]),
    "opf_session_output": (C.c_int32, [C.c_void_p, C.c_char_p, C.POINTER(opf_view)]),
    "opf_session_stats": (C.c_int32, [C.c_void_p, C.POINTER(C.c_void_p)]),
    "opf_session_trace": (C.c_int32, [C.c_void_p, C.POINTER(C.c_void_p)]),
    "opf_session_schedule_dump": (C.c_int32, [C.c_void_p, C.POINTER(C.c_void_p)]),
    "opf_dry_run": (C.c_int32, [C.c_void_p, C.c_void_p, C.c_char_p, C.c_char_p, C.c_int64,
                                C.c_int32, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p)]),
    "opf_dry_run_custom": (C.c_int32, [C.c_void_p, C.c_void_p, C.c_char_p, C.c_char_p,
                                       SCHEDULE_FN, C.c_void_p, C.c_int64,
                                       C.POINTER(C.c_void_p), C.POINTER(C.c_void_p)]),
    "opf_sched_split": (C.c_int32, [C.c_void_p, C.POINTER(C.c_int64), C.c_int32]),
    "opf_sched_ready": (C.c_int32, [C.c_void_p, C.c_int32, C.POINTER(opf_handle), C.c_int32,
                                    C.POINTER(C.c_int32)]),
    "opf_sched_handle": (C.c_int32, [C.c_void_p, C.c_int32, C.c_int32, C.POINTER(opf_handle)]),
    "opf_sched_execute": (C.c_int32, [C.c_void_p, C.POINTER(opf_handle), C.c_int32, C.c_int32,
                                      C.c_char_p]),
    "opf_sched_rows": (C.c_int32, [C.c_void_p, C.POINTER(C.c_int64)]),
    "opf_sched_num_subgraphs": (C.c_int32, [C.c_void_p, C.POINTER(C.c_int32)]),
    "opf_sched_label": (C.c_int32, [C.c_void_p, C.c_int32, C.c_char_p, C.c_int32]),
    "opf_sched_unfinished": (C.c_int32, [C.c_void_p, C.POINTER(C.c_int32)]),
}

_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                f"g.build()'` (no CPU fallback exists for the device path)")
        _lib = C.CDLL(str(LIB_PATH), mode=os.RTLD_NOW | C.RTLD_GLOBAL)
        for name, (res, args) in _SIGS.items():
            if os.environ.get("OPF_LIB") and not hasattr(_lib, name):
                continue  # an older A/B variant build may predate a symbol
            fn = getattr(_lib, name)
            fn.restype = res
            fn.argtypes = args
    return _lib


def take_string(ptr: C.c_void_p) -> str:
    s = C.cast(ptr, C.c_char_p).value.decode()
    lib().opf_free_string(ptr)
    return s
