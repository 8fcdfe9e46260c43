"""ctypes binding of the C-ABI in include/fmm_b200.h (lib/libfmm_b200.so).

The library is built in-tree by ``make -C paper_1203_0889_b200/csrc`` (or
``__graft_entry__.build()``). There is no fallback: importing the product API without the
built library raises ``LibraryMissing``.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FMM_B200_LIB") or os.path.join(HERE, "lib", "libfmm_b200.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "fmm_b200.h")

FMM_MAX_ORDER = 10
FMM_MAX_LEVEL = 21

# fmm_status
OK = 0
ERR_EMPTY_INPUT = 1
ERR_NCRIT = 2
ERR_ORDER = 3
ERR_LEVEL_OVERFLOW = 4
ERR_SINGULAR_M2L = 5
ERR_SINGULAR_EVAL = 6
ERR_CANNOT_SPLIT = 7
ERR_THETA = 8
ERR_UNSUPPORTED = 20
ERR_ARG = 21
ERR_STATE = 22
ERR_CUDA = 30
ERR_NO_DEVICE = 31
ERR_OOM = 32

PREC_FP64 = 0
PREC_FP32_P2P = 1


class LibraryMissing(RuntimeError):
    pass


class Config(C.Structure):
    _fields_ = [("order", C.c_int), ("n_crit", C.c_int), ("theta", C.c_double),
                ("mutual", C.c_int), ("precision", C.c_int), ("device", C.c_int),
                ("with_acc", C.c_int)]


class TreeInfo(C.Structure):
    _fields_ = [("nbodies", C.c_int64), ("ncells", C.c_int64), ("nleaves", C.c_int64),
                ("depth", C.c_int32), ("center", C.c_double * 3), ("half_side", C.c_double),
                ("n_m2l", C.c_int64), ("n_p2p", C.c_int64), ("p2p_body_pairs", C.c_int64),
                ("level_start", C.c_int32 * (FMM_MAX_LEVEL + 2)), ("mutual", C.c_int32),
                ("n_m2l_exec", C.c_int64), ("n_p2p_exec", C.c_int64)]


class StageTimes(C.Structure):
    _fields_ = [("build_ms", C.c_float), ("traverse_ms", C.c_float), ("upward_ms", C.c_float),
                ("m2l_ms", C.c_float), ("p2p_ms", C.c_float), ("downward_ms", C.c_float),
                ("total_ms", C.c_float), ("p2p_kernel_ms", C.c_float),
                ("m2l_kernel_ms", C.c_float), ("p2p_launches", C.c_int32),
                ("m2l_launches", C.c_int32), ("kernel_launches", C.c_int32),
                ("exchange_ms", C.c_float)]


class TraceRow(C.Structure):
    _fields_ = [("task_id", C.c_int32), ("worker_id", C.c_int32), ("kind", C.c_char * 16),
                ("start_ns", C.c_int64), ("end_ns", C.c_int64)]


class ShardInfo(C.Structure):
    _fields_ = [("rank", C.c_int32), ("world", C.c_int32), ("body_begin", C.c_int64),
                ("body_end", C.c_int64), ("own_leaves", C.c_int64), ("own_cells", C.c_int64),
                ("chunk_doubles", C.c_int64)]


_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)
_u64p = C.POINTER(C.c_uint64)
_dp = C.POINTER(C.c_double)
_vp = C.c_void_p

# name -> (restype, argtypes); every symbol declared in include/fmm_b200.h
SIGNATURES = {
    "fmm_create": (C.c_int, [C.POINTER(Config), C.POINTER(_vp)]),
    "fmm_destroy": (None, [_vp]),
    "fmm_last_error": (C.c_char_p, [_vp]),
    "fmm_version": (C.c_char_p, []),
    "fmm_set_bodies": (C.c_int, [_vp, _dp, C.c_int64]),
    "fmm_set_bodies_device": (C.c_int, [_vp, _vp, C.c_int64]),
    "fmm_build_tree": (C.c_int, [_vp]),
    "fmm_traverse": (C.c_int, [_vp]),
    "fmm_upward": (C.c_int, [_vp]),
    "fmm_m2l": (C.c_int, [_vp]),
    "fmm_p2p": (C.c_int, [_vp]),
    "fmm_downward": (C.c_int, [_vp]),
    "fmm_evaluate": (C.c_int, [_vp]),
    "fmm_synchronize": (C.c_int, [_vp]),
    "fmm_set_overlap": (C.c_int, [_vp, C.c_int]),
    "fmm_set_mutual": (C.c_int, [_vp, C.c_int]),
    "fmm_set_traversal_debug": (C.c_int, [_vp, C.c_int, C.c_int64]),
    "fmm_set_p2p_shape": (C.c_int, [_vp, C.c_int]),
    "fmm_get_traversal_regrows": (C.c_int, [_vp, C.POINTER(C.c_int)]),
    "fmm_update_bodies": (C.c_int, [_vp, _dp, C.c_int64]),
    "fmm_evaluate_reuse": (C.c_int, [_vp, C.POINTER(C.c_int)]),
    "fmm_get_stage_trace": (C.c_int, [_vp, _vp, C.c_int, C.POINTER(C.c_int)]),
    "fmm_get_results": (C.c_int, [_vp, _dp, _dp, C.c_int]),
    "fmm_results_device": (C.c_int, [_vp, C.POINTER(_vp), C.POINTER(_vp)]),
    "fmm_get_tree_info": (C.c_int, [_vp, C.POINTER(TreeInfo)]),
    "fmm_get_stage_times": (C.c_int, [_vp, C.POINTER(StageTimes)]),
    "fmm_get_cells": (C.c_int, [_vp, _i32p, _u64p, _dp, _dp, _i32p, _i32p, _i32p, _i32p, _i32p]),
    "fmm_get_permutation": (C.c_int, [_vp, _i64p]),
    "fmm_get_lists": (C.c_int, [_vp, _i64p, _i32p, _i64p, _i32p]),
    "fmm_get_expansions": (C.c_int, [_vp, _dp, _dp]),
    "fmm_load_tree": (C.c_int, [_vp, C.c_int64, _i32p, _u64p, _dp, _dp, _i32p, _i32p, _i32p,
                                _i32p, _i32p, _i64p]),
    "fmm_load_lists": (C.c_int, [_vp, C.c_int64, _i32p, C.c_int64, _i32p]),
    "fmm_load_multipoles": (C.c_int, [_vp, _dp]),
    "fmm_reset_accumulators": (C.c_int, [_vp]),
    "fmm_op_p2m": (C.c_int, [C.c_int, C.c_int64, _i32p, _dp, _dp, _dp]),
    "fmm_op_m2m": (C.c_int, [C.c_int, C.c_int64, _dp, _dp, _dp]),
    "fmm_op_m2l": (C.c_int, [C.c_int, C.c_int64, _dp, _dp, _dp]),
    "fmm_op_l2l": (C.c_int, [C.c_int, C.c_int64, _dp, _dp, _dp]),
    "fmm_op_l2p": (C.c_int, [C.c_int, C.c_int64, _i32p, _dp, _dp, _dp, _dp, _dp]),
    "fmm_op_p2p": (C.c_int, [C.c_int64, _i32p, _dp, C.c_int, _dp, _dp]),
    "fmm_op_evaluate_multipole": (C.c_int, [C.c_int, C.c_int64, _dp, _dp, _dp, _dp]),
    "fmm_op_laplace_derivatives": (C.c_int, [C.c_int, C.c_int64, _dp, _dp]),
    "fmm_op_compute_bounds": (C.c_int, [_dp, C.c_int64, _dp, _dp]),
    "fmm_op_morton_key": (C.c_int, [C.c_int64, _dp, _dp, C.c_double, C.c_int, _u64p]),
    "fmm_op_mac": (C.c_int, [C.c_int64, _dp, _dp, _dp, _dp, C.c_double, _i32p]),
    "fmm_generate_bodies": (C.c_int, [C.c_int, C.c_int64, C.c_uint64, _dp]),
    "fmm_set_partition": (C.c_int, [_vp, C.c_int, C.c_int]),
    "fmm_get_shard_info": (C.c_int, [_vp, C.POINTER(ShardInfo)]),
    "fmm_upward_local": (C.c_int, [_vp, _vp]),
    "fmm_upward_finish": (C.c_int, [_vp, _vp]),
    "fmm_set_stream": (C.c_int, [_vp, _vp]),
    "fmm_plan_partition": (C.c_int, [C.c_int64, _i32p, _i32p, _i32p, _dp, C.c_int, _i64p, _i32p]),
    "fmm_comm_unique_id": (C.c_int, [_vp]),
    "fmm_comm_init": (C.c_int, [_vp, _vp, C.c_int, C.c_int]),
    "fmm_comm_destroy": (C.c_int, [_vp]),
    "fmm_set_bodies_shard": (C.c_int, [_vp, _dp, C.c_int64, C.c_int64]),
    "fmm_evaluate_sharded": (C.c_int, [_vp, C.POINTER(ShardInfo)]),
    "fmm_get_owned_results": (C.c_int, [_vp, _dp, _dp, _i64p]),
    "fmm_set_allgather": (C.c_int, [_vp, _vp, _vp]),
}
# fmm_allgather_fn(d_send, d_recv, count, stream, user) -> int
ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p)
COMM_ID_BYTES = 128

_lib = None


def load() -> C.CDLL:
    """Load lib/libfmm_b200.so (raises LibraryMissing when it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise LibraryMissing(
            f"{LIB_PATH} is missing: build it with `make -C paper_1203_0889_b200/csrc` "
            "(the B200 path has no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib
