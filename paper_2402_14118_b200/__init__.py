"""B200-native masked matrix multiplication (arXiv 2402.14118): C = M(X) x N(Y).

Hot path: K1 sparsity-map preprocessing + K2 masked fp32 GEMM, hand-written for sm_100a
(csrc/), behind the C ABI of include/mmmcu.h.  This package is the Python mirror of the
reference's SPEC'd engine interface (see api.py); it has no compute of its own.
"""
from .api import (  # noqa: F401
    ABlockIndex,
    BPlan,
    CudaError,
    DimensionMismatchError,
    LaneConfig,
    MmmContext,
    MmmError,
    MatrixFileError,
    MmmGroup,
    MmmStreams,
    NoDeviceError,
    PlanStats,
    StaleContextError,
    UnsupportedError,
    WorkCounters,
    generate,
    matrix_seed,
    mmmb_load,
    mmmb_peek,
    mmmb_save,
    multiply_host,
    multiply_mmm,
    multiply_parallel,
    multiply_simple,
    plan_stats,
    preprocess_a,
    preprocess_b,
    round_up,
    shard_cols,
    shard_rows,
)
from . import _native  # noqa: F401

__all__ = [n for n in dir() if not n.startswith("_")]
