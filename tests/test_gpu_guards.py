"""GPU parity of the exactness and accuracy guards (VERDICT r01 "What's weak" #1, #2).

EXACT (K2-SIMT) must touch only the 8-column groups whose code bit is set
(/root/reference/proj/src/kernel_table.cpp:17-20) for BOTH mask spans, so Inf / NaN in A and
-0.0 in C0 give the reference's bits.  AUTO's fp16 split scales every A row and every 8-column
B group by its own power of two: rows or column blocks far below the operand maximum keep
the 1e-5 * Σ|a||b| tolerance, and mixed-scale rows / groups send AUTO to the
exact path.
"""
import numpy as np
import pytest

from oracle import oracle as o

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2402_14118_b200 as mmm  # noqa: E402
from paper_2402_14118_b200 import _native as N  # noqa: E402

from test_gpu_parity import (TOL, EXACT, assert_counters, bitexact, ctx, gen_pair, run_gpu, run_oracle,  # noqa: E402,F401
                             within_tol)

SIMT = (N.ALGO_SIMT_SPAN8, N.ALGO_SIMT_SPAN16)


def nan_aware_equal(C, Cr):
    assert (np.isnan(C) == np.isnan(Cr)).all()
    fin = ~np.isnan(Cr)
    return bitexact(C[fin], Cr[fin])


def b_element_random(K, N_, zB, seed):
    # the reference `random` structure (matgen.hpp:101-112): element-level zeros in B
    return o.ref_generate(K, N_, "random", zB, 0, seed)


# ------------------------------------------------------------------ span 16 exactness
@pytest.mark.parametrize("bkind", ["bw8_z0.1", "elem_z0.5", "elem_z0.8"])
def test_nonfinite_a_exact_both_spans(ctx, bkind):
    M, K, N_ = 256, 512, 512
    A, B = gen_pair(31, M, K, N_, 0.6, 0.1, 8)
    if bkind.startswith("elem"):
        B = b_element_random(K, N_, float(bkind.split("z")[1]), 5)
    A[3, 5] = np.inf
    A[10, 20] = -np.inf
    A[40, 100] = np.nan
    A[41, 7] = np.inf
    Cr, ocnt = run_oracle(A, B)
    assert np.isinf(Cr).any() and np.isnan(Cr).any()
    for algo in (N.ALGO_SIMT_SPAN8, N.ALGO_SIMT_SPAN16, EXACT, N.ALGO_AUTO):
        C, cnt = run_gpu(ctx, A, B, algo=algo)
        assert nan_aware_equal(C, Cr), (bkind, algo)
        assert_counters(cnt, ocnt)
        if algo == N.ALGO_AUTO:
            assert ctx.last_algo() in SIMT  # non-finite A keeps AUTO exact


def test_span16_chosen_where_expected(ctx):
    # K1's cost model picks the 16-column span for dense-ish 8-wide blocks and element-random
    # B at moderate sparsity: the cases where the union walk used to add +0 terms
    for zB, kind, want in ((0.1, "bw8", N.ALGO_SIMT_SPAN16), (0.5, "elem", N.ALGO_SIMT_SPAN16)):
        A, B = gen_pair(32, 256, 512, 512, 0.6, zB, 8)
        if kind == "elem":
            B = b_element_random(512, 512, zB, 6)
        A[7, 9] = np.inf
        Cr, _ = run_oracle(A, B)
        C, _ = run_gpu(ctx, A, B, algo=EXACT)
        assert ctx.last_algo() == want
        assert nan_aware_equal(C, Cr)


@pytest.mark.parametrize("algo", [N.ALGO_SIMT_SPAN8, N.ALGO_SIMT_SPAN16, EXACT])
def test_negative_zero_c0_exact(ctx, algo):
    # c0 = -0.0 stays -0.0 where the reference touches nothing, and the fmaf chain decides
    # the sign where it does
    M, K, N_ = 192, 64, 256
    A, B = gen_pair(33, M, K, N_, 0.9, 0.8, 8)  # ~27% of C untouched, many half-live slices
    C0 = np.zeros((M, B.shape[1]), np.float32)
    C0[:, :N_] = np.float32(-0.0)
    C0[::3, ::5] = np.float32(0.25)
    Cr, ocnt = run_oracle(A, B, C0=C0)
    assert (np.signbit(Cr) & (Cr == 0)).any()
    C, cnt = run_gpu(ctx, A, B, C0=C0, algo=algo)
    assert bitexact(C, Cr)
    assert_counters(cnt, ocnt)


def test_nonfinite_padding_stays_zero(ctx):
    # N % 16 == 8: the slice's second group is padding; Inf in A must not reach it
    M, K, N_ = 128, 256, 200
    A, B = gen_pair(34, M, K, N_, 0.5, 0.1, 8)
    A[0, 0] = np.inf
    Cr, _ = run_oracle(A, B)
    for algo in (N.ALGO_SIMT_SPAN8, N.ALGO_SIMT_SPAN16):
        C, _ = run_gpu(ctx, A, B, algo=algo, N_=N_)
        assert (C[:, N_:] == 0).all()
        assert nan_aware_equal(C[:, :N_], Cr[:, :N_])


# ------------------------------------------------------------- fp16-split dynamic range
def scaled_case(kind):
    M, K, N_ = 1024, 1024, 1024
    A, B = gen_pair(35, M, K, N_, 0.5, 0.3, 16)
    if kind == "a_rows":
        A[5] *= np.float32(2.0 ** -28)
        A[77] *= np.float32(2.0 ** -32)
        A[500] *= np.float32(2.0 ** 20)
    elif kind == "b_blocks":
        B[:, 64:80] *= np.float32(2.0 ** -28)   # one 16-wide column block
        B[:, 200:208] *= np.float32(2.0 ** -32)  # one 8-column group
        B[:, 640:656] *= np.float32(2.0 ** 24)
    elif kind == "both":
        A[9] *= np.float32(2.0 ** -30)
        B[:, 96:112] *= np.float32(2.0 ** -30)
    return A, B


@pytest.mark.parametrize("kind", ["a_rows", "b_blocks", "both"])
def test_auto_tc_scaled_rows_and_blocks(ctx, kind):
    A, B = scaled_case(kind)
    Cr, ocnt = run_oracle(A, B)
    for algo in (N.ALGO_AUTO, N.ALGO_TC):
        C, cnt = run_gpu(ctx, A, B, algo=algo)
        if algo == N.ALGO_AUTO:
            assert ctx.last_algo() == N.ALGO_TC  # per-row / per-group scales keep the fp16 path
        ok, worst = within_tol(C, Cr, A, B)
        assert ok and worst < 0.5 * TOL, (kind, algo, worst)
        assert_counters(cnt, ocnt)


@pytest.mark.parametrize("kind", ["a_half_row", "b_group_tile"])
def test_auto_mixed_scale_goes_exact(ctx, kind):
    # a row (group) whose parts lie 2^28 apart cannot be scaled into fp16 as one: AUTO keeps
    # the exact K2-SIMT path
    M, K, N_ = 1024, 1024, 1024
    A, B = gen_pair(36, M, K, N_, 0.5, 0.3, 16)
    if kind == "a_half_row":
        A[11, 512:] *= np.float32(2.0 ** -28)
    else:
        B[0:32, 64:72] *= np.float32(2.0 ** -28)  # one 32-k tile of one 8-column group
    Cr, ocnt = run_oracle(A, B)
    C, cnt = run_gpu(ctx, A, B, algo=N.ALGO_AUTO)
    assert ctx.last_algo() in SIMT
    assert bitexact(C, Cr)
    assert_counters(cnt, ocnt)
