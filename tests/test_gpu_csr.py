"""K2-CSR (k2_csr.cuh): the multiply driven by A's non-zeros, bit-exact against the
oracle like K2-SIMT, on the shapes it is built for (very sparse / skinny A, BASELINE configs[3])
and on the edge cases of the exact path (ragged shapes, accumulate, Inf / NaN, -0.0)."""
import numpy as np
import pytest

from oracle import oracle as o

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2402_14118_b200 import _native as N  # noqa: E402
from paper_2402_14118_b200.api import VALUE_NORMAL, VALUE_RELU  # noqa: E402

from test_gpu_parity import (assert_counters, bitexact, ctx, gen_pair, run_gpu, run_oracle,  # noqa: E402,F401
                             within_tol)
from test_gpu_guards import nan_aware_equal  # noqa: E402

CSR = N.ALGO_CSR


@pytest.mark.parametrize("M,K,N_,zA,zB,bw", [(1024, 1024, 1024, 0.8, 0.8, 16), (100, 77, 130, 0.6, 0.6, 8),
                                             (257, 1000, 600, 0.95, 0.5, 32), (1, 5, 1, 0.0, 0.0, 8),
                                             (129, 65, 257, 0.5, 0.9, 8), (64, 4096, 2048, 0.95, 0.85, 16)])
def test_csr_bitexact(ctx, M, K, N_, zA, zB, bw):
    A, B = gen_pair(61, M, K, N_, zA, zB, bw)
    rng = np.random.default_rng(M + K)
    C0 = np.zeros((M, B.shape[1]), np.float32)
    C0[:, :N_] = rng.uniform(-1, 1, (M, N_)).astype(np.float32)
    C, cnt = run_gpu(ctx, A, B, C0=C0, algo=CSR, N_=N_)
    Cr, ocnt = run_oracle(A, B, C0=C0)
    assert bitexact(C, Cr)
    assert (C[:, N_:] == 0).all()
    assert_counters(cnt, ocnt)


def test_csr_nonfinite_and_negzero(ctx):
    M, K, N_ = 192, 320, 256
    A, B = gen_pair(62, M, K, N_, 0.9, 0.5, 8)
    A[3, 5] = np.inf
    A[40, 100] = np.nan
    C0 = np.zeros((M, B.shape[1]), np.float32)
    C0[:, :N_] = np.float32(-0.0)
    Cr, _ = run_oracle(A, B, C0=C0)
    C, _ = run_gpu(ctx, A, B, C0=C0, algo=CSR)
    assert nan_aware_equal(C, Cr)
    fin = ~np.isnan(Cr)
    assert (np.signbit(C[fin]) == np.signbit(Cr[fin])).all()


def test_csr_cfg4(ctx):
    # BASELINE configs[3]: 64 x 12288 x 49152, A ReLU ~95% zeros, B 16-wide blocks kept 0.15
    A, B = gen_pair(4, 64, 12288, 49152, 0.0, 0.85, 16, a_kind=VALUE_RELU, a_thresh=1.6448536269514722,
                    b_kind=VALUE_NORMAL, b_sigma=0.02)
    Cr, ocnt = run_oracle(A, B)
    C, cnt = run_gpu(ctx, A, B, algo=CSR)
    assert bitexact(C, Cr)
    assert_counters(cnt, ocnt)


@pytest.mark.parametrize("zA,zB,bw", [(0.95, 0.95, 8), (0.9, 0.9, 16), (0.6, 0.8, 32)])
def test_csr_sweep_cells(ctx, zA, zB, bw):
    A, B = gen_pair(63, 4096, 4096, 4096, zA, zB, bw)
    C, cnt = run_gpu(ctx, A, B, algo=CSR)
    Cr, ocnt = run_oracle(A, B)
    assert bitexact(C, Cr)
    assert_counters(cnt, ocnt)
