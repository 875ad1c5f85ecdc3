"""Python handle on the CPU ORACLE (oracle/mmm_oracle.c) and on the compiled reference
(oracle/_ref/libmmmref.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference leg, always as the checker or the timed CPU baseline —
never by the product package.  See the header of mmm_oracle.c for the reference file:line
each function restates, and DESIGN.md "Oracle" for how it is pinned.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from ctypes import POINTER, c_double, c_int, c_int64, c_uint32, c_uint64, c_void_p

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORC_SO = os.path.join(HERE, "_build", "liborc.so")
REF_SO = os.path.join(HERE, "_ref", "libmmmref.so")
REF_SO_V4 = os.path.join(HERE, "_ref", "libmmmref_v4.so")  # -march=x86-64-v4 (AVX-512) build


def _cpu_has_avx512() -> bool:
    try:
        flags = open("/proc/cpuinfo").read()
    except OSError:
        return False
    return all(f in flags for f in (" avx512f", " avx512bw", " avx512dq", " avx512vl"))


def ref_so_path() -> str:
    """The reference build for this host: the AVX-512 one where the CPU has it (what the
    reference's own -march=native gives there), else the AVX2 one."""
    return REF_SO_V4 if (os.path.exists(REF_SO_V4) and _cpu_has_avx512()) else REF_SO

STRUCTURES = {"random": 0, "block_random": 1, "column": 2, "block_column": 3}


class OrcCounters(ctypes.Structure):
    _fields_ = [("kernel_invocations", c_uint64), ("lane_fma_ops", c_uint64), ("rows_skipped", c_uint64),
                ("regions_skipped_by_zero_code", c_uint64)]


class RefCounters(ctypes.Structure):
    _fields_ = [("kernel_invocations", c_uint64), ("lane_fma_ops", c_uint64), ("rows_skipped", c_uint64),
                ("regions_skipped_by_zero_code", c_uint64), ("preprocess_ns", c_int64), ("multiply_ns", c_int64)]


_orc = None
_ref = None


def _ensure_built(path: str, target: str):
    if not os.path.exists(path):
        subprocess.run(["make", "-C", HERE] + ([target] if target else []), check=True,
                       stdout=subprocess.DEVNULL)


def lib():
    global _orc
    if _orc is None:
        _ensure_built(ORC_SO, "")
        L = ctypes.CDLL(ORC_SO)
        L.orc_mix64.restype = c_uint64
        L.orc_mix64.argtypes = [c_uint64]
        L.orc_hash_coords.restype = c_uint64
        L.orc_hash_coords.argtypes = [c_uint64] * 4
        L.orc_unit_double.restype = c_double
        L.orc_unit_double.argtypes = [c_uint64]
        L.orc_ref_generate.restype = c_int
        L.orc_ref_generate.argtypes = [c_void_p, c_int64, c_int64, c_int64, c_int, c_double, c_int64, c_uint64,
                                       c_int64, c_int64]
        L.orc_gen_iid.restype = c_int
        L.orc_gen_iid.argtypes = [c_void_p, c_int64, c_int64, c_int64, c_uint64, c_int, c_double, c_double, c_int,
                                  c_double, c_int64]
        L.orc_gen_iid_rows.restype = c_int
        L.orc_gen_iid_rows.argtypes = [c_void_p, c_int64, c_int64, c_int64, c_int64, c_uint64, c_int, c_double,
                                       c_double, c_int, c_double, c_int64]
        L.orc_region_fma.restype = c_int
        L.orc_region_fma.argtypes = [c_uint32, c_int, c_int, c_void_p, ctypes.c_float, c_void_p]
        L.orc_pattern_codes.restype = c_int
        L.orc_pattern_codes.argtypes = [c_void_p, c_int64, c_int64, c_int, c_int, c_void_p]
        L.orc_bplan_order.restype = c_int
        L.orc_bplan_order.argtypes = [c_void_p, c_int64, c_int64, c_int64, c_int64, c_void_p, c_void_p]
        L.orc_plan_stats.restype = None
        L.orc_plan_stats.argtypes = [c_void_p, c_int64, POINTER(c_int64), POINTER(c_double), POINTER(c_double)]
        L.orc_ablock_index.restype = c_int64
        L.orc_ablock_index.argtypes = [c_void_p, c_int64, c_int64, c_int64, c_int64, c_void_p, c_void_p]
        L.orc_a_bitmap.restype = None
        L.orc_a_bitmap.argtypes = [c_void_p, c_int64, c_int64, c_int64, c_void_p]
        L.orc_a_csr.restype = c_int64
        L.orc_a_csr.argtypes = [c_void_p, c_int64, c_int64, c_int64, c_void_p, c_void_p]
        L.orc_multiply_simple.restype = None
        L.orc_multiply_simple.argtypes = [c_void_p, c_int64, c_void_p, c_int64, c_void_p, c_int64, c_int64, c_int64,
                                          c_int64]
        L.orc_multiply_mmm.restype = c_int
        L.orc_multiply_mmm.argtypes = [c_void_p, c_int64, c_void_p, c_int64, c_void_p, c_int64, c_int64, c_int64,
                                       c_int64, c_void_p, c_int, c_int, POINTER(OrcCounters)]
        L.orc_bruteforce_lane_ops.restype = c_uint64
        L.orc_region_fma_f64.argtypes = [c_uint32, c_int, c_int, c_void_p, c_double, c_void_p]
        L.orc_pattern_codes_f64.argtypes = [c_void_p, c_int64, c_int64, c_int, c_int, c_void_p]
        L.orc_multiply_simple_f64.argtypes = [c_void_p, c_int64, c_void_p, c_int64, c_void_p, c_int64, c_int64,
                                              c_int64, c_int64]
        L.orc_multiply_simple_f64.restype = None
        L.orc_multiply_mmm_f64.argtypes = [c_void_p, c_int64, c_void_p, c_int64, c_void_p, c_int64, c_int64, c_int64,
                                           c_int64, c_void_p, c_int, c_int, c_void_p]
        L.orc_bruteforce_lane_ops.argtypes = [c_void_p, c_int64, c_void_p, c_int64, c_int64, c_int64, c_int]
        L.orc_check_tolerance.restype = c_int64
        L.orc_check_tolerance.argtypes = [c_void_p, c_void_p, c_int64, c_void_p, c_int64, c_void_p, c_int64, c_int64,
                                          c_int64, c_int64, c_void_p, c_int64, c_double, POINTER(c_double)]
        L.orc_num_threads.restype = c_int
        _orc = L
    return _orc


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref_lib():
    """The reference's own compiled code (kernel_table.cpp, matrix_io.cpp, matgen.hpp)."""
    global _ref
    if _ref is None:
        if not ref_available():
            raise FileNotFoundError(f"{REF_SO} not built (needs /root/reference at build time)")
        L = ctypes.CDLL(ref_so_path())
        L.ref_generate_f32.restype = c_int
        L.ref_generate_f32.argtypes = [c_int64, c_int64, c_int, c_double, c_int64, c_uint64, c_int, c_int, c_int,
                                       c_void_p, POINTER(c_int64)]
        L.ref_kernel_apply_f32.restype = c_int
        L.ref_kernel_apply_f32.argtypes = [c_int, c_int, c_int, c_uint32, c_void_p, ctypes.c_float, c_void_p]
        L.ref_write_matrix_f32.restype = c_int
        L.ref_write_matrix_f32.argtypes = [c_void_p, c_int64, c_int64, c_int64, ctypes.c_char_p]
        L.ref_read_matrix_f32.restype = c_int
        L.ref_read_matrix_f32.argtypes = [ctypes.c_char_p, c_void_p, c_int64, c_int64, c_int64]
        L.ref_multiply_parallel_f32.restype = c_int
        L.ref_multiply_parallel_f32.argtypes = [c_void_p, c_int64, c_void_p, c_int64, c_void_p, c_int64, c_int64,
                                                c_int64, c_int64, c_int64, c_int64, c_int, POINTER(RefCounters)]
        L.ref_multiply_mmm_f32.restype = c_int
        L.ref_multiply_mmm_f32.argtypes = [c_void_p, c_int64, c_void_p, c_int64, c_void_p, c_int64, c_int64, c_int64,
                                           c_int64, c_int64, c_int, POINTER(RefCounters)]
        L.ref_kernel_apply_f64.restype = c_int
        L.ref_kernel_apply_f64.argtypes = [c_int, c_int, c_int, c_uint32, c_void_p, c_double, c_void_p]
        for nm in ("ref_multiply_lane_f32", "ref_multiply_lane_f64"):
            f = getattr(L, nm)
            f.restype = c_int
            f.argtypes = [c_void_p, c_int64, c_void_p, c_int64, c_void_p, c_int64, c_int64, c_int64, c_int, c_int,
                          c_int, POINTER(RefCounters)]
        L.ref_max_threads.restype = c_int
        _ref = L
    return _ref


def _p(a: np.ndarray):
    return a.ctypes.data


def num_threads() -> int:
    return lib().orc_num_threads()


# ------------------------------------------------------------------------ generators
def ref_generate(rows, cols, structure="random", target=0.0, block_len=0, seed=0, lane=(8, 8, 1)):
    """Oracle restatement of generate<float> (matgen.hpp:77-148); returns padded array."""
    R = lane[0] * lane[1] * lane[2]
    ld = (cols + R - 1) // R * R
    out = np.zeros((rows, ld), dtype=np.float32)
    st = lib().orc_ref_generate(_p(out), rows, cols, ld, STRUCTURES[structure], target, block_len, seed, R, lane[0])
    if st != 0:
        raise ValueError("invalid generator arguments")
    return out


def gen_iid(rows, cols, seed, value_kind=0, sigma=1.0, thresh=0.0, mask_kind=0, p=0.0, block=1, ld=None, row0=0):
    ld = cols if ld is None else ld
    out = np.zeros((rows, ld), dtype=np.float32)
    if lib().orc_gen_iid_rows(_p(out), rows, cols, ld, row0, seed, value_kind, sigma, thresh, mask_kind, p,
                              block) != 0:
        raise ValueError("invalid generator arguments")
    return out


# ------------------------------------------------------------------------------ plans
def pattern_codes(B: np.ndarray, group_width=8, pattern_bits=8) -> np.ndarray:
    """Codes [K][ld/R] of an f32 or f64 B (dtype kept)."""
    f64 = B.dtype == np.float64
    B = np.ascontiguousarray(B, dtype=np.float64 if f64 else np.float32)
    K, ld = B.shape
    R = group_width * pattern_bits
    codes = np.zeros((K, ld // R), dtype=np.uint32)
    fn = lib().orc_pattern_codes_f64 if f64 else lib().orc_pattern_codes
    if fn(_p(B), K, ld, group_width, pattern_bits, _p(codes)) != 0:
        raise ValueError("ld must be a multiple of the region width")
    return codes


def bplans(codes: np.ndarray, region_width=64, leaf_dim=256):
    K, nreg = codes.shape
    codes = np.ascontiguousarray(codes, dtype=np.uint32)
    rpl = leaf_dim // region_width
    n_pl = ((K + leaf_dim - 1) // leaf_dim) * ((nreg + rpl - 1) // rpl)
    plans = np.zeros(K * nreg, dtype=np.uint32)
    off = np.zeros(n_pl + 1, dtype=np.int64)
    if lib().orc_bplan_order(_p(codes), K, nreg, region_width, leaf_dim, _p(plans), _p(off)) != 0:
        raise ValueError("leaf_dim must be a multiple of the region width")
    return [plans[off[i]:off[i + 1]] for i in range(n_pl)]


def plan_stats(codes: np.ndarray):
    c = np.ascontiguousarray(codes, dtype=np.uint32).ravel()
    n, z, m = c_int64(), c_double(), c_double()
    lib().orc_plan_stats(_p(c), c.size, ctypes.byref(n), ctypes.byref(z), ctypes.byref(m))
    return n.value, z.value, m.value


def ablock_index(A: np.ndarray, K=None, block_dim=256):
    A = np.ascontiguousarray(A, dtype=np.float32)
    M, lda = A.shape
    K = lda if K is None else K
    nseg = M * ((K + 7) // 8)
    counts = np.zeros(nseg, dtype=np.uint8)
    offsets = np.zeros((nseg, 8), dtype=np.uint8)
    n = lib().orc_ablock_index(_p(A), M, K, lda, block_dim, _p(counts), _p(offsets))
    assert n == nseg
    return counts, offsets


def a_bitmap(A: np.ndarray, K=None):
    A = np.ascontiguousarray(A, dtype=np.float32)
    M, lda = A.shape
    K = lda if K is None else K
    bits = np.zeros((M, (K + 31) // 32), dtype=np.uint32)
    lib().orc_a_bitmap(_p(A), M, K, lda, _p(bits))
    return bits


def a_csr(A: np.ndarray, K=None):
    A = np.ascontiguousarray(A, dtype=np.float32)
    M, lda = A.shape
    K = lda if K is None else K
    row_ptr = np.zeros(M + 1, dtype=np.int64)
    nnz = lib().orc_a_csr(_p(A), M, K, lda, _p(row_ptr), None)
    cols = np.zeros(max(nnz, 1), dtype=np.uint32)
    lib().orc_a_csr(_p(A), M, K, lda, _p(row_ptr), _p(cols))
    return row_ptr, cols[:nnz]


# ----------------------------------------------------------------------------- engine
def region_fma(code, c, a, b, group_width=8, pattern_bits=8):
    f64 = np.asarray(c).dtype == np.float64
    dt = np.float64 if f64 else np.float32
    c = np.ascontiguousarray(c, dtype=dt)
    b = np.ascontiguousarray(b, dtype=dt)
    fn = lib().orc_region_fma_f64 if f64 else lib().orc_region_fma
    if fn(code, group_width, pattern_bits, _p(c), float(a), _p(b)) != 0:
        raise ValueError("bad pattern size")
    return c


def multiply_simple(C, A, B):
    """In-place C += A @ B, i-k-j fmaf."""
    M, K = A.shape
    N = C.shape[1]
    fn = lib().orc_multiply_simple_f64 if C.dtype == np.float64 else lib().orc_multiply_simple
    fn(_p(C), C.shape[1], _p(A), A.shape[1], _p(B), B.shape[1], M, K, N)
    return C


def multiply_mmm(C, A, B, K=None, N=None, group_width=8, pattern_bits=8, codes=None):
    """In-place C += A @ B over the masks; returns the WorkCounters dict.

    A is M x lda (logical K columns), B is K x ldb with ldb a multiple of the region
    width, C is M x ldc with ldc >= ldb (padding columns included)."""
    M, lda = A.shape
    Kb, ldb = B.shape
    K = Kb if K is None else K
    N = ldb if N is None else N
    if codes is None:
        codes = pattern_codes(B, group_width, pattern_bits)
    codes = np.ascontiguousarray(codes, dtype=np.uint32)
    cnt = OrcCounters()
    fn = lib().orc_multiply_mmm_f64 if C.dtype == np.float64 else lib().orc_multiply_mmm
    st = fn(_p(C), C.shape[1], _p(A), lda, _p(B), ldb, M, K, N, _p(codes), group_width, pattern_bits,
            ctypes.byref(cnt))
    if st != 0:
        raise ValueError("bad multiply arguments")
    return {k: int(getattr(cnt, k)) for k, _ in OrcCounters._fields_}


def bruteforce_lane_ops(A, B, group_width=8):
    M, lda = A.shape
    K, ldb = B.shape
    return int(lib().orc_bruteforce_lane_ops(_p(A), lda, _p(B), ldb, M, K, group_width))


def check_tolerance(Cg, Cr, A, B, rows=None, tol=1e-5):
    """|Cg - Cr| <= tol * Σ|a||b| (fp64 denominators).  Returns (n_bad, max_ratio)."""
    M, lda = A.shape
    K, ldb = B.shape
    N = Cg.shape[1]
    mr = c_double()
    if rows is not None:
        rows = np.ascontiguousarray(rows, dtype=np.int64)
        bad = lib().orc_check_tolerance(_p(Cg), _p(Cr), Cg.shape[1], _p(A), lda, _p(B), ldb, M, K, N, _p(rows),
                                        rows.size, tol, ctypes.byref(mr))
    else:
        bad = lib().orc_check_tolerance(_p(Cg), _p(Cr), Cg.shape[1], _p(A), lda, _p(B), ldb, M, K, N, None, 0, tol,
                                        ctypes.byref(mr))
    return int(bad), mr.value


# ----------------------------------------------------------------- reference (compiled)
def ref_generate_compiled(rows, cols, structure="random", target=0.0, block_len=0, seed=0, lane=(8, 8, 1)):
    L = ref_lib()
    pc = c_int64()
    st = L.ref_generate_f32(rows, cols, STRUCTURES[structure], target, block_len, seed, *lane, None, ctypes.byref(pc))
    if st != 0:
        raise ValueError(f"reference generate failed with status {st}")
    out = np.zeros((rows, pc.value), dtype=np.float32)
    L.ref_generate_f32(rows, cols, STRUCTURES[structure], target, block_len, seed, *lane, _p(out), ctypes.byref(pc))
    return out


def ref_kernel_apply(code, c, a, b, lane=(8, 8, 1)):
    c = np.ascontiguousarray(c, dtype=np.float32).copy()
    b = np.ascontiguousarray(b, dtype=np.float32)
    st = ref_lib().ref_kernel_apply_f32(*lane, code, _p(c), a, _p(b))
    return st, c


def ref_kernel_apply_f64(code, c, a, b, lane=(4, 8, 1)):
    c = np.ascontiguousarray(c, dtype=np.float64).copy()
    b = np.ascontiguousarray(b, dtype=np.float64)
    st = ref_lib().ref_kernel_apply_f64(lane[0], lane[1], lane[2], code, _p(c), float(a), _p(b))
    return st, c


def ref_multiply_lane(C, A, B, lane):
    """The reference KernelTable<T> (f32 / f64 by C's dtype) for any lane config: C += A*B over
    the P-bit codes (Fig. 4 A-skip); returns the counters (golden fixtures only)."""
    M, lda = A.shape
    K, ldb = B.shape
    cnt = RefCounters()
    fn = ref_lib().ref_multiply_lane_f64 if C.dtype == np.float64 else ref_lib().ref_multiply_lane_f32
    st = fn(_p(C), C.shape[1], _p(A), lda, _p(B), ldb, M, K, lane[0], lane[1], lane[2], ctypes.byref(cnt))
    if st != 0:
        raise RuntimeError(f"reference multiply failed with status {st}")
    return {k: int(getattr(cnt, k)) for k, _ in RefCounters._fields_}


def ref_multiply_mmm(C, A, B, row0=0, row1=None, workers=0):
    """The reference-kind CPU baseline: SPEC preprocess_b / preprocess_a (ABlockIndex) and the
    leaf-blocked multiply over the reference's compiled KernelTable (ref_driver.cpp)."""
    M, lda = A.shape
    K, ldb = B.shape
    row1 = M if row1 is None else row1
    cnt = RefCounters()
    st = ref_lib().ref_multiply_mmm_f32(_p(C), C.shape[1], _p(A), lda, _p(B), ldb, K, ldb, row0, row1, workers,
                                        ctypes.byref(cnt))
    if st != 0:
        raise RuntimeError(f"reference multiply failed with status {st}")
    return {k: int(getattr(cnt, k)) for k, _ in RefCounters._fields_}


def ref_multiply_parallel(C, A, B, row0=0, row1=None, workers=0):
    M, lda = A.shape
    K, ldb = B.shape
    row1 = M if row1 is None else row1
    cnt = RefCounters()
    st = ref_lib().ref_multiply_parallel_f32(_p(C), C.shape[1], _p(A), lda, _p(B), ldb, M, K, ldb, row0, row1,
                                             workers, ctypes.byref(cnt))
    if st != 0:
        raise RuntimeError(f"reference multiply failed with status {st}")
    return {k: int(getattr(cnt, k)) for k, _ in RefCounters._fields_}
