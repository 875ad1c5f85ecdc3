"""ctypes binding of the C ABI in include/mmmcu.h (libmmmcu.so, built in-tree).

The product path is the CUDA library only: if the shared object is missing or cannot be
loaded this module raises; there is no Python or CPU fallback for any computation.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_double, c_int, c_int32, c_int64, c_uint8, c_uint32, c_uint64, c_void_p

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MMMCU_LIB") or os.path.join(_HERE, "_lib", "libmmmcu.so")

# mmmcu_status
OK = 0
ERR_INVALID_ARG = 1
ERR_DIM_MISMATCH = 2
ERR_STALE = 3
ERR_UNSUPPORTED = 4
ERR_CUDA = 5
ERR_NOT_READY = 6
ERR_OVERFLOW = 7
ERR_WORKERS = 8
ERR_NO_DEVICE = 9
ERR_FILE_IO = 10
ERR_FILE_FORMAT = 11
ERR_FILE_TRUNCATED = 12

# mmmcu_dtype (matrix.hpp:13-26)
F32 = 0
F64 = 1

# mmmcu_algo
ALGO_AUTO = 0
ALGO_SIMT_BCAST = 1
ALGO_DENSE = 2
ALGO_SIMT_SPAN8 = 3
ALGO_SIMT_SPAN16 = 4
ALGO_TC = 5
ALGO_TC32 = 6
ALGO_CSR = 7


class Lane(ctypes.Structure):
    _fields_ = [("w", c_int32), ("p", c_int32), ("v", c_int32)]


class Counters(ctypes.Structure):
    _fields_ = [
        ("kernel_invocations", c_uint64),
        ("lane_fma_ops", c_uint64),
        ("rows_skipped", c_uint64),
        ("regions_skipped_by_zero_code", c_uint64),
    ]


class PlanStatsC(ctypes.Structure):
    _fields_ = [("region_count", c_int64), ("zero_region_fraction", c_double), ("mean_popcount", c_double)]


# (name, restype, argtypes) of every symbol include/mmmcu.h declares
SIGNATURES = [
    ("mmmcu_abi_version", c_int, []),
    ("mmmcu_last_error", c_char_p, [c_void_p]),
    ("mmmcu_ctx_create", c_int, [c_int, POINTER(c_void_p)]),
    ("mmmcu_ctx_destroy", c_int, [c_void_p]),
    ("mmmcu_set_stream", c_int, [c_void_p, c_void_p]),
    ("mmmcu_validate_lane", c_int, [c_void_p, Lane]),
    ("mmmcu_preprocess", c_int, [c_void_p, c_void_p, c_int64, c_int64, c_int64, c_void_p, c_int64, c_int64, Lane,
                                 c_uint64, c_uint64]),
    ("mmmcu_preprocess_a", c_int, [c_void_p, c_void_p, c_int64, c_int64, c_int64, c_uint64]),
    ("mmmcu_preprocess_b", c_int, [c_void_p, c_void_p, c_int64, c_int64, c_int64, Lane, c_uint64]),
    ("mmmcu_get_counters", c_int, [c_void_p, POINTER(Counters)]),
    ("mmmcu_get_plan_stats", c_int, [c_void_p, POINTER(PlanStatsC)]),
    ("mmmcu_export_b_codes", c_int, [c_void_p, c_void_p, c_int64]),
    ("mmmcu_export_bplans", c_int, [c_void_p, c_int64, c_void_p, c_int64, c_void_p, c_int64, POINTER(c_int64)]),
    ("mmmcu_export_a_bitmap", c_int, [c_void_p, c_void_p, c_int64]),
    ("mmmcu_export_a_csr", c_int, [c_void_p, c_void_p, c_void_p, c_int64, POINTER(c_int64)]),
    ("mmmcu_export_ablock_index", c_int, [c_void_p, c_int64, c_void_p, c_int64, c_void_p, c_int64,
                                          POINTER(c_int64)]),
    ("mmmcu_multiply", c_int, [c_void_p, c_void_p, c_int64, c_void_p, c_void_p, c_uint64, c_uint64,
                               POINTER(Counters)]),
    ("mmmcu_multiply_parallel", c_int, [c_void_p, c_void_p, c_int64, c_void_p, c_void_p, c_uint64, c_uint64, c_int,
                                        POINTER(Counters)]),
    ("mmmcu_set_algo", c_int, [c_void_p, c_int]),
    ("mmmcu_last_algo", c_int, [c_void_p, POINTER(c_int)]),
    ("mmmcu_multiply_simple", c_int, [c_void_p, c_void_p, c_int64, c_void_p, c_int64, c_void_p, c_int64, c_int64,
                                      c_int64, c_int64]),
    ("mmmcu_multiply_host", c_int, [c_void_p, c_void_p, c_int64, c_void_p, c_int64, c_void_p, c_int64, c_int64,
                                    c_int64, c_int64, POINTER(Counters)]),
    ("mmmcu_generate", c_int, [c_void_p, c_void_p, c_int64, c_int64, c_int64, c_int64, c_uint64, c_int, c_double,
                               c_double,
                               c_int, c_double, c_int64]),
    ("mmmcu_shard_rows", c_int, [c_int64, c_int, c_int, POINTER(c_int64), POINTER(c_int64)]),
    ("mmmcu_shard_cols", c_int, [c_int64, c_int, c_int, POINTER(c_int64), POINTER(c_int64)]),
    ("mmmcu_io_last_error", c_char_p, []),
    ("mmmcu_mmmb_peek", c_int, [c_char_p, POINTER(c_int32), POINTER(c_int64), POINTER(c_int64)]),
    ("mmmcu_mmmb_load", c_int, [c_char_p, c_void_p, c_int64, c_int64, c_void_p, POINTER(c_int64), POINTER(c_int64)]),
    ("mmmcu_mmmb_save", c_int, [c_char_p, c_void_p, c_int64, c_int64, c_int64, c_void_p]),
    ("mmmcu_group_create", c_int, [c_int, POINTER(c_int), POINTER(c_void_p)]),
    ("mmmcu_group_destroy", c_int, [c_void_p]),
    ("mmmcu_group_last_error", c_char_p, [c_void_p]),
    ("mmmcu_group_size", c_int, [c_void_p]),
    ("mmmcu_group_uses_nccl", c_int, [c_void_p]),
    ("mmmcu_group_ctx", c_void_p, [c_void_p, c_int]),
    ("mmmcu_group_set_algo", c_int, [c_void_p, c_int]),
    ("mmmcu_multiply_sharded", c_int, [c_void_p, POINTER(c_void_p), c_int64, POINTER(c_void_p), c_int64, c_void_p,
                                       c_int64, c_int64, c_int64, c_int64, c_uint64, c_uint64, POINTER(Counters),
                                       POINTER(c_double)]),
    ("mmmcu_multiply_sharded_cols", c_int, [c_void_p, POINTER(c_void_p), c_int64, c_void_p, c_int64, c_void_p,
                                            c_int64, c_int64, c_int64, c_int64, c_uint64, c_uint64, POINTER(Counters),
                                            POINTER(c_double)]),
    ("mmmcu_preprocess_host", c_int, [c_void_p, c_void_p, c_int64, c_int64, c_int64, c_void_p, c_int64, c_int64, Lane,
                                      c_uint64, c_uint64]),
    ("mmmcu_multiply_planned_host", c_int, [c_void_p, c_void_p, c_int64, c_uint64, c_uint64, c_int,
                                            POINTER(Counters)]),
    # every dtype / lane config (kgen.cuh)
    ("mmmcu_validate_lane_t", c_int, [c_void_p, c_int, Lane]),
    ("mmmcu_preprocess_a_t", c_int, [c_void_p, c_int, c_void_p, c_int64, c_int64, c_int64, c_uint64]),
    ("mmmcu_preprocess_b_t", c_int, [c_void_p, c_int, c_void_p, c_int64, c_int64, c_int64, Lane, c_uint64]),
    ("mmmcu_preprocess_t", c_int, [c_void_p, c_int, c_void_p, c_int64, c_int64, c_int64, c_void_p, c_int64, c_int64,
                                   Lane, c_uint64, c_uint64]),
    ("mmmcu_multiply_t", c_int, [c_void_p, c_int, c_void_p, c_int64, c_void_p, c_void_p, c_uint64, c_uint64,
                                 POINTER(Counters)]),
    ("mmmcu_multiply_simple_t", c_int, [c_void_p, c_int, c_void_p, c_int64, c_void_p, c_int64, c_void_p, c_int64,
                                        c_int64, c_int64, c_int64]),
    ("mmmcu_export_b_codes16", c_int, [c_void_p, c_void_p, c_int64]),
    ("mmmcu_export_bplans16", c_int, [c_void_p, c_int64, c_void_p, c_int64, c_void_p, c_int64, POINTER(c_int64)]),
    ("mmmcu_plan_info", c_int, [c_void_p, POINTER(c_int), POINTER(Lane)]),
    ("mmmcu_multiply_host_t", c_int, [c_void_p, c_int, c_void_p, c_int64, c_void_p, c_int64, c_void_p, c_int64,
                                      c_int64, c_int64, c_int64, Lane, POINTER(Counters)]),
    ("mmmcu_preprocess_host_t", c_int, [c_void_p, c_int, c_void_p, c_int64, c_int64, c_int64, c_void_p, c_int64,
                                        c_int64, Lane, c_uint64, c_uint64]),
    ("mmmcu_multiply_simple_host_t", c_int, [c_void_p, c_int, c_void_p, c_int64, c_void_p, c_int64, c_void_p,
                                             c_int64, c_int64, c_int64, c_int64]),
    ("mmmcu_multiply_planned_host_t", c_int, [c_void_p, c_int, c_void_p, c_int64, c_uint64, c_uint64, c_int,
                                              POINTER(Counters)]),
]

_lib = None


def load() -> ctypes.CDLL:
    """Load libmmmcu.so (fails loudly when it was not built: no fallback exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the masked multiply has no CPU fallback)"
        )
    lib = ctypes.CDLL(LIB_PATH)
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib
