"""Python mirror of the reference's hot-path interface over the C ABI (include/mmmcu.h).

Names, argument meaning and error behaviour follow the SPEC'd C++ engine of the reference
 so tests read like the reference's own acceptance list:

    LaneConfig            matrix.hpp:31-44
    WorkCounters
    BPlan / ABlockIndex
    preprocess_b          SPEC.md:196-205     -> list[BPlan]
    preprocess_a          SPEC.md:206-214     -> ABlockIndex
    plan_stats
    MmmContext            SPEC.md:248-251     (device plans + staleness tags)
    multiply_mmm          SPEC.md:276-284     -> WorkCounters
    multiply_parallel     SPEC.md:285-293     -> WorkCounters
    multiply_simple

Operands are CUDA float32 torch tensors (device memory and streams only: torch is the
plumbing) in the reference Matrix layout — row-major, unit column stride, leading dimension
= stride(0).  torch's in-place version counter (`Tensor._version`) plays the role of
Matrix::version() (matrix.hpp:115): mutating an operand after preprocessing makes the
context stale, exactly as SPEC.md:280 requires.  Host numpy operands go through
mmmcu_multiply_host (copies inside the library).  Every computation runs in the CUDA
library; nothing here computes on the CPU.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _native as N


# ----------------------------------------------------------------------------- errors
class MmmError(RuntimeError):
    """Base class of library failures."""


class DimensionMismatchError(ValueError):
    """a.cols != b.rows or c has the wrong shape."""


class StaleContextError(MmmError):
    """the context's plans do not belong to these operands any more."""


class UnsupportedError(MmmError):
    """Lane config / dtype without a GPU kernel (no CPU fallback exists)."""


class CudaError(MmmError):
    pass


class MatrixFileError(MmmError):
    """MatrixFileError family of matrix_io.hpp:15-29 (MMMB files)."""


class BadFormatError(MatrixFileError):
    """BadMagicError / UnknownDtypeError / unsupported version."""


class TruncatedFileError(MatrixFileError):
    pass


class FileIoError(MatrixFileError):
    pass


class NoDeviceError(MmmError):
    pass


def _raise(status: int, msg: str):
    if status == N.ERR_INVALID_ARG:
        raise ValueError(msg)  # std::invalid_argument
    if status == N.ERR_DIM_MISMATCH:
        raise DimensionMismatchError(msg)
    if status == N.ERR_STALE:
        raise StaleContextError(msg)
    if status == N.ERR_UNSUPPORTED:
        raise UnsupportedError(msg)
    if status == N.ERR_OVERFLOW:
        raise OverflowError(msg)  # std::overflow_error
    if status == N.ERR_WORKERS:
        raise ValueError(msg)  # SPEC.md:290 worker_count == 0 rejected
    if status == N.ERR_NO_DEVICE:
        raise NoDeviceError(msg)
    if status == N.ERR_FILE_IO:
        raise FileIoError(msg)
    if status == N.ERR_FILE_FORMAT:
        raise BadFormatError(msg)
    if status == N.ERR_FILE_TRUNCATED:
        raise TruncatedFileError(msg)
    if status == N.ERR_NOT_READY:
        raise MmmError(msg)
    raise CudaError(msg)


# ------------------------------------------------------------------------------ types
@dataclass(frozen=True)
class LaneConfig:
    """LaneConfig (matrix.hpp:31-44); f32 default {8, 8, 1} => region width 64."""

    w: int = 8
    p: int = 8
    v: int = 1

    def group_width(self) -> int:
        return self.w * self.v

    def region_width(self) -> int:
        return self.w * self.p * self.v

    def _c(self) -> N.Lane:
        return N.Lane(self.w, self.p, self.v)


@dataclass
class WorkCounters:
    """WorkCounters."""

    kernel_invocations: int = 0
    lane_fma_ops: int = 0
    rows_skipped: int = 0
    regions_skipped_by_zero_code: int = 0

    @staticmethod
    def _from(c: N.Counters) -> "WorkCounters":
        return WorkCounters(int(c.kernel_invocations), int(c.lane_fma_ops), int(c.rows_skipped),
                            int(c.regions_skipped_by_zero_code))


@dataclass
class BPlan:
    """BPlan: codes of one leaf sub-block in multiply order."""

    submatrix_id: int
    codes: np.ndarray  # uint8 (P = 8)


@dataclass
class ABlockIndex:
    """ABlockIndex (layout decision SPEC.md:229): block-major segments."""

    block_dim: int
    counts: np.ndarray  # uint8 [n_segments]
    offsets: np.ndarray  # uint8 [n_segments, 8], 0xFF in unused slots


@dataclass
class PlanStats:
    region_count: int
    zero_region_fraction: float
    mean_popcount: float


def round_up(x: int, m: int) -> int:
    return (x + m - 1) // m * m


# --------------------------------------------------------------------------- helpers
def _lib():
    return N.load()


def _check_tensor(t, name: str):
    return _check_tensor_t(t, name)[:2]


def _check_tensor_t(t, name: str):
    """(pointer, leading dimension, mmmcu_dtype) of a CUDA float32 / float64 row-major tensor
    (Dtype::f32 / f64, matrix.hpp:13-26)."""
    import torch

    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name} must be a torch.Tensor (CUDA float32 / float64) or use the *_host entry points")
    if t.dtype not in (torch.float32, torch.float64):
        raise UnsupportedError(f"{name}: only float32 / float64 operands have a GPU kernel (got {t.dtype})")
    if not t.is_cuda:
        raise ValueError(f"{name} must live on a CUDA device")
    if t.dim() != 2 or t.stride(1) != 1:
        raise ValueError(f"{name} must be a row-major 2-D tensor with unit column stride")
    return t.data_ptr(), int(t.stride(0)), (N.F64 if t.dtype == torch.float64 else N.F32)


def _version(t) -> int:
    # Matrix::version() analogue: storage pointer + in-place modification counter
    return (int(t._version) << 1) ^ (t.data_ptr() << 20)


class MmmContext:
    """MmmContext: device plans of one (A, B) pair on one GPU.

    Owns a native context (mmmcu_ctx): bitmaps, index lists, pattern codes, counters and
    all scratch.  Work is enqueued on the torch stream current at call time.
    """

    def __init__(self, device: int = 0, lane: LaneConfig = LaneConfig(), leaf_dim: int = 256):
        lib = _lib()
        h = ctypes.c_void_p()
        st = lib.mmmcu_ctx_create(int(device), ctypes.byref(h))
        if st != N.OK:
            _raise(st, lib.mmmcu_last_error(None).decode())
        self._h = h
        self.device = int(device)
        self.lane = lane
        self.leaf_dim = int(leaf_dim)
        self._shape = None  # (M, K, N)
        self.counters = WorkCounters()

    # -- plumbing
    def _check(self, status: int):
        if status != N.OK:
            _raise(status, _lib().mmmcu_last_error(self._h).decode())

    def _sync_stream(self):
        import torch

        s = torch.cuda.current_stream(self.device)
        self._check(_lib().mmmcu_set_stream(self._h, ctypes.c_void_p(s.cuda_stream)))

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            _lib().mmmcu_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_algo(self, algo: int):
        self._check(_lib().mmmcu_set_algo(self._h, int(algo)))

    def last_algo(self) -> int:
        v = ctypes.c_int()
        self._check(_lib().mmmcu_last_algo(self._h, ctypes.byref(v)))
        return v.value

    # -- plans
    def preprocess(self, a, b):
        """preprocess_a(a) + preprocess_b(b) on the device (one K1 pass over each)."""
        pa, lda, dta = _check_tensor_t(a, "a")
        pb, ldb, dtb = _check_tensor_t(b, "b")
        M, K = a.shape
        Kb, Nn = b.shape
        if K != Kb:
            raise DimensionMismatchError(f"a.cols ({K}) != b.rows ({Kb})")
        if dta != dtb:
            raise ValueError("a and b must have the same dtype")
        self._sync_stream()
        self._check(_lib().mmmcu_preprocess_t(self._h, dta, pa, M, K, lda, pb, Nn, ldb, self.lane._c(), _version(a),
                                              _version(b)))
        self._shape = (M, K, Nn)
        return self

    def preprocess_a_only(self, a):
        pa, lda, dt = _check_tensor_t(a, "a")
        self._sync_stream()
        self._check(_lib().mmmcu_preprocess_a_t(self._h, dt, pa, a.shape[0], a.shape[1], lda, _version(a)))

    def preprocess_b_only(self, b):
        pb, ldb, dt = _check_tensor_t(b, "b")
        self._sync_stream()
        self._check(_lib().mmmcu_preprocess_b_t(self._h, dt, pb, b.shape[0], b.shape[1], ldb, self.lane._c(),
                                                _version(b)))

    def planned_counters(self) -> WorkCounters:
        c = N.Counters()
        self._check(_lib().mmmcu_get_counters(self._h, ctypes.byref(c)))
        return WorkCounters._from(c)

    def plan_stats(self) -> PlanStats:
        s = N.PlanStatsC()
        self._check(_lib().mmmcu_get_plan_stats(self._h, ctypes.byref(s)))
        return PlanStats(int(s.region_count), float(s.zero_region_fraction), float(s.mean_popcount))

    # -- exports of the canonical formats
    def export_b_codes(self, K: int, ldb: int) -> np.ndarray:
        """Pattern codes [K][ldb / R] of the current plan: uint8 for P <= 8, else uint16."""
        R = self.lane.region_width()
        out = np.empty((K, ldb // R), dtype=np.uint16)
        self._check(_lib().mmmcu_export_b_codes16(self._h, out.ctypes.data, out.size))
        return out.astype(np.uint8) if self.lane.p <= 8 else out

    def export_bplans(self, K: int, ldb: int, leaf_dim: Optional[int] = None) -> List[BPlan]:
        leaf = self.leaf_dim if leaf_dim is None else int(leaf_dim)
        R = self.lane.region_width()
        nreg = ldb // R
        rpl = max(leaf // R, 1)
        n_pl = ((K + leaf - 1) // leaf) * ((nreg + rpl - 1) // rpl)
        plans = np.empty(K * nreg, dtype=np.uint16)
        off = np.empty(n_pl + 1, dtype=np.int64)
        n = ctypes.c_int64()
        self._check(_lib().mmmcu_export_bplans16(self._h, leaf, plans.ctypes.data, plans.size, off.ctypes.data,
                                                 off.size, ctypes.byref(n)))
        if self.lane.p <= 8:
            plans = plans.astype(np.uint8)
        return [BPlan(p, plans[off[p]:off[p + 1]].copy()) for p in range(n.value)]

    def export_a_bitmap(self, M: int, K: int) -> np.ndarray:
        out = np.empty((M, (K + 31) // 32), dtype=np.uint32)
        self._check(_lib().mmmcu_export_a_bitmap(self._h, out.ctypes.data, out.size))
        return out

    def export_a_csr(self, M: int):
        row_ptr = np.empty(M + 1, dtype=np.int64)
        nnz = ctypes.c_int64()
        self._check(_lib().mmmcu_export_a_csr(self._h, row_ptr.ctypes.data, None, 0, ctypes.byref(nnz)))
        cols = np.empty(max(nnz.value, 1), dtype=np.uint32)
        self._check(_lib().mmmcu_export_a_csr(self._h, row_ptr.ctypes.data, cols.ctypes.data, cols.size,
                                              ctypes.byref(nnz)))
        return row_ptr, cols[: nnz.value]

    def export_ablock_index(self, M: int, K: int, block_dim: int = 256) -> ABlockIndex:
        nseg = M * ((K + 7) // 8)
        counts = np.empty(nseg, dtype=np.uint8)
        offsets = np.empty((nseg, 8), dtype=np.uint8)
        n = ctypes.c_int64()
        self._check(_lib().mmmcu_export_ablock_index(self._h, block_dim, counts.ctypes.data, counts.size,
                                                     offsets.ctypes.data, offsets.size, ctypes.byref(n)))
        return ABlockIndex(block_dim, counts, offsets)

    # -- multiply
    def multiply(self, c, a, b, want_counters: bool = True) -> Optional[WorkCounters]:
        pc, ldc, dt = _check_tensor_t(c, "c")
        pa, _, _ = _check_tensor_t(a, "a")
        pb, _, _ = _check_tensor_t(b, "b")
        if self._shape is not None and (c.shape[0] != a.shape[0] or c.shape[1] != b.shape[1]):
            raise DimensionMismatchError(f"c is {tuple(c.shape)}, expected ({a.shape[0]}, {b.shape[1]})")
        self._sync_stream()
        cnt = N.Counters()
        self._check(_lib().mmmcu_multiply_t(self._h, dt, pc, ldc, pa, pb, _version(a), _version(b),
                                            ctypes.byref(cnt) if want_counters else None))
        if want_counters:
            self.counters = WorkCounters._from(cnt)
            return self.counters
        return None


# ------------------------------------------------------------------ SPEC entry points
def _ctx_for(t, ctx: Optional[MmmContext], lane: LaneConfig) -> MmmContext:
    if ctx is not None:
        return ctx
    return MmmContext(device=t.device.index or 0, lane=lane)


def preprocess_b(b, lane: LaneConfig = LaneConfig(), leaf_dim: int = 256, ctx: Optional[MmmContext] = None
                 ) -> List[BPlan]:
    """preprocess_b: one BPlan per leaf_dim x leaf_dim sub-block of B."""
    c = _ctx_for(b, ctx, lane)
    c.lane = lane
    c.preprocess_b_only(b)
    return c.export_bplans(b.shape[0], b.stride(0), leaf_dim)


def preprocess_a(a, block_dim: int = 256, ctx: Optional[MmmContext] = None) -> ABlockIndex:
    """preprocess_a: blocked-sparse-row index of A."""
    c = _ctx_for(a, ctx, LaneConfig())
    c.preprocess_a_only(a)
    return c.export_ablock_index(a.shape[0], a.shape[1], block_dim)


def plan_stats(plans: List[BPlan], pattern_bits: int = 8) -> PlanStats:
    """plan_stats over exported plans (a pure summary of their codes)."""
    if not plans:
        return PlanStats(0, 0.0, 0.0)
    codes = np.concatenate([p.codes for p in plans]).astype(np.uint32)
    n = int(codes.size)
    pop = int(np.unpackbits(codes.astype(np.uint8)[:, None], axis=1).sum()) if pattern_bits <= 8 else int(
        sum(bin(int(x)).count("1") for x in codes))
    return PlanStats(n, float((codes == 0).sum()) / n if n else 0.0, pop / n if n else 0.0)


def multiply_mmm(context: MmmContext, c, a, b) -> WorkCounters:
    """multiply_mmm: c += a*b over the context's masks; exact counters."""
    return context.multiply(c, a, b)


def multiply_parallel(context: MmmContext, c, a, b, worker_count: int) -> WorkCounters:
    """multiply_parallel: worker_count == 0 rejected; same result bits."""
    pc, ldc, dt = _check_tensor_t(c, "c")
    pa, _, _ = _check_tensor_t(a, "a")
    pb, _, _ = _check_tensor_t(b, "b")
    if dt == N.F64:  # the typed path: the worker count is validated, then the same multiply
        if int(worker_count) <= 0:
            _raise(N.ERR_WORKERS, "worker_count must be positive")
        return context.multiply(c, a, b)
    context._sync_stream()
    cnt = N.Counters()
    context._check(_lib().mmmcu_multiply_parallel(context._h, pc, ldc, pa, pb, _version(a), _version(b),
                                                  int(worker_count), ctypes.byref(cnt)))
    context.counters = WorkCounters._from(cnt)
    return context.counters


def multiply_simple(c, a, b, ctx: Optional[MmmContext] = None) -> None:
    """multiply_simple: dense i-k-j c += a*b (fma per term) on the GPU."""
    pc, ldc, dt = _check_tensor_t(c, "c")
    pa, lda, _ = _check_tensor_t(a, "a")
    pb, ldb, _ = _check_tensor_t(b, "b")
    M, K = a.shape
    Kb, Nn = b.shape
    if K != Kb or c.shape[0] != M or c.shape[1] != Nn:
        raise DimensionMismatchError(f"shapes a{tuple(a.shape)} b{tuple(b.shape)} c{tuple(c.shape)}")
    cx = _ctx_for(a, ctx, LaneConfig())
    cx._sync_stream()
    cx._check(_lib().mmmcu_multiply_simple_t(cx._h, dt, pc, ldc, pa, lda, pb, ldb, M, K, Nn))


def multiply_host(c: np.ndarray, a: np.ndarray, b: np.ndarray, ctx: Optional[MmmContext] = None) -> WorkCounters:
    """Host-operand path (mmmcu_multiply_host): H2D, K1, K2, D2H inside the library."""
    for name, t in (("a", a), ("b", b), ("c", c)):
        if t.dtype != np.float32 or t.ndim != 2 or not t.flags.c_contiguous:
            raise ValueError(f"{name} must be a C-contiguous float32 2-D array")
    M, K = a.shape
    Kb, Nn = b.shape
    if K != Kb or c.shape != (M, Nn):
        raise DimensionMismatchError(f"shapes a{a.shape} b{b.shape} c{c.shape}")
    cx = ctx if ctx is not None else MmmContext()
    cnt = N.Counters()
    cx._check(_lib().mmmcu_multiply_host(cx._h, c.ctypes.data, c.shape[1], a.ctypes.data, a.shape[1], b.ctypes.data,
                                         b.shape[1], M, K, Nn, ctypes.byref(cnt)))
    return WorkCounters._from(cnt)


# ------------------------------------------------------------------- synthetic inputs
VALUE_UNIFORM, VALUE_NORMAL, VALUE_RELU = 0, 1, 2
MASK_NONE, MASK_ELEMENT, MASK_BLOCK = 0, 1, 2


def generate(out, seed: int, value_kind: int = VALUE_UNIFORM, sigma: float = 1.0, thresh: float = 0.0,
             mask_kind: int = MASK_NONE, p: float = 0.0, block: int = 1, cols: Optional[int] = None,
             row0: int = 0, ctx: Optional[MmmContext] = None):
    """Fill a CUDA float32 tensor with the seeded i.i.d. generator (mmmcu_generate)."""
    po, ld = _check_tensor(out, "out")
    cx = _ctx_for(out, ctx, LaneConfig())
    cx._sync_stream()
    cx._check(_lib().mmmcu_generate(cx._h, po, out.shape[0], out.shape[1] if cols is None else cols, ld, int(row0),
                                    ctypes.c_uint64(seed & 0xFFFFFFFFFFFFFFFF), value_kind, sigma, thresh,
                                    mask_kind, p, block))
    return out


def shard_rows(M: int, world: int, rank: int):
    """Row partition of a sharded multiply: rank owns [row0, row1)."""
    r0, r1 = ctypes.c_int64(), ctypes.c_int64()
    st = _lib().mmmcu_shard_rows(M, world, rank, ctypes.byref(r0), ctypes.byref(r1))
    if st != N.OK:
        _raise(st, _lib().mmmcu_last_error(None).decode())
    return r0.value, r1.value


# ------------------------------------------------------------------ MMMB files (f3)
def mmmb_peek(path: str):
    """(dtype, rows, cols) of an MMMB file (peek_dtype, matrix_io.hpp:37-38); no device needed."""
    d, r, c = ctypes.c_int32(), ctypes.c_int64(), ctypes.c_int64()
    st = _lib().mmmcu_mmmb_peek(str(path).encode(), ctypes.byref(d), ctypes.byref(r), ctypes.byref(c))
    if st != N.OK:
        _raise(st, _lib().mmmcu_io_last_error().decode())
    return {0: "f32", 1: "f64"}[d.value], r.value, c.value


def mmmb_load(path: str, device: int = 0, lane: LaneConfig = LaneConfig()):
    """read_matrix<float> (matrix_io.hpp:42-48) into device memory: a CUDA tensor with the
    Matrix padding (ld = round_up(cols, region width), padding zero); returns the logical view."""
    import torch

    _, rows, cols = mmmb_peek(path)
    ld = round_up(cols, lane.region_width())
    t = torch.empty((rows, ld), dtype=torch.float32, device=f"cuda:{device}")
    r, c = ctypes.c_int64(), ctypes.c_int64()
    st = _lib().mmmcu_mmmb_load(str(path).encode(), t.data_ptr(), ld, rows,
                                ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream), ctypes.byref(r),
                                ctypes.byref(c))
    if st != N.OK:
        _raise(st, _lib().mmmcu_io_last_error().decode())
    return t[:, :cols]


def mmmb_save(path: str, t) -> None:
    """write_matrix (matrix_io.hpp:32-33) of a CUDA float32 matrix (logical columns only)."""
    import torch

    p, ld = _check_tensor(t, "t")
    st = _lib().mmmcu_mmmb_save(str(path).encode(), p, t.shape[0], t.shape[1], ld,
                                ctypes.c_void_p(torch.cuda.current_stream(t.device).cuda_stream))
    if st != N.OK:
        _raise(st, _lib().mmmcu_io_last_error().decode())


def shard_cols(Ncols: int, world: int, rank: int):
    """Column partition for skinny A (SURVEY.md §8(e) "Other shapes"): whole 64-column regions."""
    c0, c1 = ctypes.c_int64(), ctypes.c_int64()
    st = _lib().mmmcu_shard_cols(Ncols, world, rank, ctypes.byref(c0), ctypes.byref(c1))
    if st != N.OK:
        _raise(st, _lib().mmmcu_last_error(None).decode())
    return c0.value, c1.value


class MmmGroup:
    """Single-process multi-GPU group (mmmcu_group_*): one context + stream per device, B (or,
    column-sharded, A) broadcast with NCCL from devices[0].  Row-sharded calls take per-rank A / C
    shards on their devices (rows shard_rows(M, g, r))."""

    def __init__(self, devices):
        lib = _lib()
        self.devices = [int(d) for d in devices]
        arr = (ctypes.c_int * len(self.devices))(*self.devices)
        h = ctypes.c_void_p()
        st = lib.mmmcu_group_create(len(self.devices), arr, ctypes.byref(h))
        if st != N.OK:
            _raise(st, lib.mmmcu_group_last_error(None).decode())
        self._h = h
        self.broadcast_ms = 0.0

    def _check(self, status: int):
        if status != N.OK:
            _raise(status, _lib().mmmcu_group_last_error(self._h).decode())

    @property
    def size(self) -> int:
        return _lib().mmmcu_group_size(self._h)

    @property
    def uses_nccl(self) -> bool:
        return bool(_lib().mmmcu_group_uses_nccl(self._h))

    def set_algo(self, algo: int):
        self._check(_lib().mmmcu_group_set_algo(self._h, int(algo)))

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            _lib().mmmcu_group_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def multiply_sharded(self, c_shards, a_shards, b, version_a: int = 0, version_b: int = 0) -> WorkCounters:
        """C_r += A_r * B for every rank r (A_r / C_r = rows shard_rows(M, g, r) on devices[r])."""
        import torch

        g = self.size
        if len(c_shards) != g or len(a_shards) != g:
            raise ValueError(f"need {g} A and C shards")
        pb, ldb = _check_tensor(b, "b")
        K, Nn = b.shape
        M = sum(int(a.shape[0]) for a in a_shards)
        lda = ldc = None
        pa, pc = [], []
        for r, (a, c) in enumerate(zip(a_shards, c_shards)):
            r0, r1 = shard_rows(M, g, r)
            if a.shape[0] != r1 - r0 or c.shape[0] != r1 - r0:
                raise DimensionMismatchError(f"shard {r} must hold rows [{r0}, {r1})")
            x, la = _check_tensor(a, "a")
            y, lc = _check_tensor(c, "c")
            if (lda is not None and la != lda) or (ldc is not None and lc != ldc):
                raise ValueError("all shards must share one leading dimension")
            lda, ldc = la, lc
            pa.append(x)
            pc.append(y)
        for d in set(self.devices):
            torch.cuda.synchronize(d)
        A = (ctypes.c_void_p * g)(*pa)
        C = (ctypes.c_void_p * g)(*pc)
        cnt, ms = N.Counters(), ctypes.c_double()
        self._check(_lib().mmmcu_multiply_sharded(self._h, C, ldc, A, lda, pb, ldb, M, K, Nn, int(version_a),
                                                  int(version_b), ctypes.byref(cnt), ctypes.byref(ms)))
        self.broadcast_ms = ms.value
        return WorkCounters._from(cnt)

    def multiply_sharded_cols(self, c_slabs, a, b, version_a: int = 0, version_b: int = 0) -> WorkCounters:
        """C[:, slab r] += A * B[:, slab r] on devices[r] (slabs shard_cols(N, g, r)); A, B on devices[0]."""
        import torch

        g = self.size
        pa, lda = _check_tensor(a, "a")
        pb, ldb = _check_tensor(b, "b")
        M, K = a.shape
        Nn = b.shape[1]
        ldc = None
        pc = []
        for r, c in enumerate(c_slabs):
            c0, c1 = shard_cols(Nn, g, r)
            y, lc = _check_tensor(c, "c")
            if c.shape[0] != M or c.shape[1] != c1 - c0:
                raise DimensionMismatchError(f"slab {r} must be {M} x {c1 - c0}")
            if ldc is not None and lc != ldc:
                raise ValueError("all slabs must share one leading dimension")
            ldc = lc
            pc.append(y)
        for d in set(self.devices):
            torch.cuda.synchronize(d)
        C = (ctypes.c_void_p * g)(*pc)
        cnt, ms = N.Counters(), ctypes.c_double()
        self._check(_lib().mmmcu_multiply_sharded_cols(self._h, C, ldc, pa, lda, pb, ldb, M, K, Nn, int(version_a),
                                                       int(version_b), ctypes.byref(cnt), ctypes.byref(ms)))
        self.broadcast_ms = ms.value
        return WorkCounters._from(cnt)


class MmmStreams:
    """Independent multiplies on n contexts, each on its own CUDA stream.

    One multiply is K1 (HBM-bound) followed by K2 (tensor-bound on the AUTO path), and K2-TC
    leaves a few SMs free (it takes the fewest CTA pairs that keep its number of rounds), so a
    batch of independent (C, A, B) jobs runs faster when the K1 chain of one job shares the GPU
    with the K2 of another (BASELINE configs[1], 75 cells: 22.9 -> 21.5 ms with 2 streams).
    Jobs are dealt round-robin; the jobs of one stream run in order, every stream owns its plans (context).
    The C operands of jobs on different streams must not alias.
    """

    def __init__(self, n: int = 2, device: int = 0, lane: LaneConfig = LaneConfig()):  # lane: the SIMD LaneConfig
        import torch

        if n < 1:
            raise ValueError("MmmStreams needs at least one stream")
        self.device = int(device)
        self.contexts = [MmmContext(self.device, lane) for _ in range(int(n))]
        self.streams = [torch.cuda.Stream(torch.device("cuda", self.device)) for _ in range(int(n))]
        self._next = 0

    def __len__(self) -> int:
        return len(self.contexts)

    def fork(self):
        """Every stream waits for the work already queued on the current stream."""
        import torch

        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(self.device))
        for st in self.streams:
            st.wait_event(ev)

    def join(self):
        """The current stream waits for every stream."""
        import torch

        cur = torch.cuda.current_stream(self.device)
        for st in self.streams:
            cur.wait_stream(st)

    def submit(self, c, a, b, stream: Optional[int] = None) -> int:
        """preprocess(a, b) + C += A*B on the next stream (or number `stream`); returns the one used."""
        import torch

        i = self._next if stream is None else int(stream) % len(self.contexts)
        if stream is None:
            self._next = (self._next + 1) % len(self.contexts)
        with torch.cuda.stream(self.streams[i]):
            self.contexts[i].preprocess(a, b)
            self.contexts[i].multiply(c, a, b, want_counters=False)
        return i

    def run(self, jobs) -> None:
        """fork(), submit every (c, a, b) of jobs round-robin, join()."""
        self.fork()
        for (c, a, b) in jobs:
            self.submit(c, a, b)
        self.join()

    def close(self):
        for cx in self.contexts:
            cx.close()


def matrix_seed(seed: int, tag: str) -> int:
    """Per-matrix seed hash_coords(seed, tag) (SURVEY.md §7 hard part 9; rng.hpp:18)."""
    def mix64(x):
        x = (x + 0x9E3779B97F4A7C15) & 0xFFFFFFFFFFFFFFFF
        x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & 0xFFFFFFFFFFFFFFFF
        x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & 0xFFFFFFFFFFFFFFFF
        return x ^ (x >> 31)

    h = mix64(seed ^ 0x7FB5D329728EA185)
    h = mix64(h ^ ord(tag[0]))
    h = mix64(h ^ 0)
    return mix64(h ^ 0)
