"""The reference-kind CPU baseline (oracle/_ref: SPEC preprocess_a / preprocess_b and the
leaf-blocked ABlockIndex multiply over the reference's compiled KernelTable, ref_driver.cpp)
computes exactly what the oracle does: C bit-identical, WorkCounters equal."""
import numpy as np
import pytest

from oracle import oracle as o

pytestmark = pytest.mark.skipif(not o.ref_available(), reason="oracle/_ref not built (needs /root/reference)")


@pytest.mark.parametrize("M,K,N,zA,zB,bw", [(300, 530, 320, 0.8, 0.8, 16), (256, 256, 256, 0.6, 0.6, 8),
                                            (513, 1030, 700, 0.95, 0.7, 32)])
def test_ref_mmm_matches_oracle(M, K, N, zA, zB, bw):
    ldb = (N + 63) // 64 * 64
    A = o.gen_iid(M, K, seed=11, mask_kind=1, p=zA)
    B = o.gen_iid(K, N, seed=12, mask_kind=2, p=zB, block=bw, ld=ldb)
    C0 = o.gen_iid(M, N, seed=13, ld=ldb)
    want = C0.copy()
    cw = o.multiply_mmm(want, A, B, K=K, N=N)
    for rows in ((0, M), (M // 3, M)):
        got = C0.copy()
        cg = o.ref_multiply_mmm(got, A, B, row0=rows[0], row1=rows[1], workers=4)
        r0, r1 = rows
        assert np.array_equal(got[r0:r1].view(np.uint32), want[r0:r1].view(np.uint32))
        assert np.array_equal(got[:r0], C0[:r0])
        if r0 == 0:
            for key in ("kernel_invocations", "lane_fma_ops", "rows_skipped", "regions_skipped_by_zero_code"):
                assert cg[key] == cw[key], key
