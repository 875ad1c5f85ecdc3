"""GPU parity of the lane-general and f64 paths (kgen.cuh) against
the CPU oracle, which tests/test_oracle_golden.py pins to the reference's KernelTable<T>
for these lanes and dtypes.

Bar: codes, BPlans, plan_stats, bitmap, CSR and WorkCounters bit-exact; C bit-identical
(the general kernel forms exactly the reference's per-element fma chain)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_2402_14118_b200 as mmm  # noqa: E402
from oracle import oracle as orc  # noqa: E402  (checker only)
from paper_2402_14118_b200 import _native as N  # noqa: E402

pytestmark = pytest.mark.gpu

LANES32 = [(1, 8, 1), (2, 8, 1), (4, 8, 1), (4, 4, 4), (8, 2, 4), (16, 4, 1), (32, 8, 2), (2, 16, 2), (1, 1, 1)]
LANES64 = [(4, 8, 1), (2, 16, 1), (8, 8, 1), (1, 4, 1), (16, 4, 4)]


def _operands(M, K, N_, lane, f64, seed, zA=0.7, zB=0.6):
    R = lane[0] * lane[1] * lane[2]
    ldb = (N_ + R - 1) // R * R
    A = orc.gen_iid(M, K, seed=seed, mask_kind=1, p=zA)
    B = orc.gen_iid(K, N_, seed=seed + 1, mask_kind=2, p=zB, block=max(1, lane[0] * lane[2]), ld=ldb)
    C0 = np.zeros((M, ldb), np.float32)
    C0[:, :N_] = orc.gen_iid(M, N_, seed=seed + 2)
    if f64:  # full f64 mantissas
        A, B, C0 = A.astype(np.float64) / 3.0, B.astype(np.float64) / 7.0, C0.astype(np.float64) / 11.0
    return A, B, C0, ldb


def _bits(x):
    return x.view(np.uint64 if x.dtype == np.float64 else np.uint32)


def _run(lane, A, B, C0, N_, algo=None):
    dev = torch.device("cuda:0")
    ctx = mmm.MmmContext(0, lane=mmm.LaneConfig(*lane))
    a = torch.from_numpy(A).to(dev)
    # the Matrix layout: B and C carry the padded leading dimension
    b = torch.from_numpy(B).to(dev)[:, :N_]
    c = torch.from_numpy(C0).to(dev)
    ctx.preprocess(a, b)
    cv = c[:, :N_]
    cnt = ctx.multiply(cv, a, b)
    torch.cuda.synchronize()
    return ctx, c.cpu().numpy(), cnt


def _check_plan(ctx, lane, A, B, K, ldb):
    G, P = lane[0] * lane[2], lane[1]
    R = G * P
    want_codes = orc.pattern_codes(B, G, P)
    got_codes = ctx.export_b_codes(K, ldb)
    assert np.array_equal(got_codes.astype(np.uint32), want_codes)
    leaf = max(R, 256 // R * R) if R <= 256 else R
    got_pl = ctx.export_bplans(K, ldb, leaf_dim=leaf)
    want_pl = orc.bplans(want_codes, region_width=R, leaf_dim=leaf)
    assert len(got_pl) == len(want_pl)
    for gp, wp in zip(got_pl, want_pl):
        assert np.array_equal(gp.codes.astype(np.uint32), wp)
    st = ctx.plan_stats()
    n, z, m = orc.plan_stats(want_codes)
    assert st.region_count == n
    assert st.zero_region_fraction == pytest.approx(z, abs=0)
    assert st.mean_popcount == pytest.approx(m, rel=1e-12)
    M = A.shape[0]
    nz = A != 0
    kw = (K + 31) // 32
    want_bits = np.zeros((M, kw), np.uint32)
    for k in range(K):
        want_bits[:, k // 32] |= nz[:, k].astype(np.uint32) << np.uint32(k % 32)
    assert np.array_equal(ctx.export_a_bitmap(M, K), want_bits)
    row_ptr, cols = ctx.export_a_csr(M)
    assert np.array_equal(row_ptr, np.concatenate([[0], np.cumsum(nz.sum(1))]))
    assert np.array_equal(cols, np.nonzero(nz)[1].astype(np.uint32))


@pytest.mark.parametrize("lane", LANES32)
def test_f32_other_lanes_bitexact(lane):
    M, K, N_ = 70, 130, 150
    A, B, C0, ldb = _operands(M, K, N_, lane, False, seed=40 + lane[0] + lane[1])
    want = C0.copy()
    cw = orc.multiply_mmm(want, A, B, K=K, N=ldb, group_width=lane[0] * lane[2], pattern_bits=lane[1])
    ctx, got, cnt = _run(lane, A, B, C0, N_)
    assert np.array_equal(_bits(got), _bits(want)), lane
    assert cnt.lane_fma_ops == cw["lane_fma_ops"] and cnt.kernel_invocations == cw["kernel_invocations"]
    assert cnt.rows_skipped == cw["rows_skipped"]
    assert cnt.regions_skipped_by_zero_code == cw["regions_skipped_by_zero_code"]
    _check_plan(ctx, lane, A, B, K, ldb)


@pytest.mark.parametrize("lane", LANES64)
def test_f64_bitexact(lane):
    M, K, N_ = 66, 140, 100
    A, B, C0, ldb = _operands(M, K, N_, lane, True, seed=90 + lane[0] + lane[1])
    want = C0.copy()
    cw = orc.multiply_mmm(want, A, B, K=K, N=ldb, group_width=lane[0] * lane[2], pattern_bits=lane[1])
    ctx, got, cnt = _run(lane, A, B, C0, N_)
    assert got.dtype == np.float64
    assert np.array_equal(_bits(got), _bits(want)), lane
    assert (cnt.lane_fma_ops, cnt.kernel_invocations, cnt.rows_skipped, cnt.regions_skipped_by_zero_code) == (
        cw["lane_fma_ops"], cw["kernel_invocations"], cw["rows_skipped"], cw["regions_skipped_by_zero_code"])
    _check_plan(ctx, lane, A, B, K, ldb)


def test_f64_bigger_and_accumulate():
    # a few hundred rows / columns, two accumulating multiplies on one plan
    lane = (4, 8, 1)
    M, K, N_ = 300, 520, 260
    A, B, C0, ldb = _operands(M, K, N_, lane, True, seed=7, zA=0.8, zB=0.8)
    want = C0.copy()
    for _ in range(2):
        orc.multiply_mmm(want, A, B, K=K, N=ldb, group_width=4, pattern_bits=8)
    dev = torch.device("cuda:0")
    ctx = mmm.MmmContext(0, lane=mmm.LaneConfig(*lane))
    a = torch.from_numpy(A).to(dev)
    bb = torch.from_numpy(B).to(dev)
    b = bb[:, :N_]
    c = torch.from_numpy(C0).to(dev)
    cv = c[:, :N_]
    ctx.preprocess(a, b)
    ctx.multiply(cv, a, b)
    mmm.multiply_parallel(ctx, cv, a, b, 4)
    torch.cuda.synchronize()
    assert np.array_equal(_bits(c.cpu().numpy()), _bits(want))
    with pytest.raises(ValueError):
        mmm.multiply_parallel(ctx, cv, a, b, 0)


def test_f64_nonfinite_and_negative_zero():
    # Inf in A: the reference only forms fma(a, b, c) for set groups; -0.0 in C0 stays -0.0
    # where nothing is added
    lane = (4, 8, 1)
    M, K, N_ = 40, 64, 96
    A, B, C0, ldb = _operands(M, K, N_, lane, True, seed=13)
    A[3, 5] = np.inf
    A[7, 9] = -np.inf
    C0[:, :N_][C0[:, :N_] > 0.05] = -0.0
    want = C0.copy()
    orc.multiply_mmm(want, A, B, K=K, N=ldb, group_width=4, pattern_bits=8)
    _, got, _ = _run(lane, A, B, C0, N_)
    nan_w, nan_g = np.isnan(want), np.isnan(got)
    assert np.array_equal(nan_w, nan_g)
    assert np.array_equal(_bits(np.where(nan_w, 0.0, got)), _bits(np.where(nan_w, 0.0, want)))


def test_f64_multiply_simple_bitexact():
    M, K, N_ = 70, 90, 110
    A = orc.gen_iid(M, K, seed=3).astype(np.float64) / 3.0
    B = orc.gen_iid(K, N_, seed=4).astype(np.float64) / 7.0
    C0 = orc.gen_iid(M, N_, seed=5).astype(np.float64)
    want = orc.multiply_simple(C0.copy(), A, B)
    dev = torch.device("cuda:0")
    c = torch.from_numpy(C0).to(dev)
    mmm.multiply_simple(c, torch.from_numpy(A).to(dev), torch.from_numpy(B).to(dev))
    torch.cuda.synchronize()
    assert np.array_equal(_bits(c.cpu().numpy()), _bits(want))


def test_general_path_errors():
    dev = torch.device("cuda:0")
    ctx = mmm.MmmContext(0, lane=mmm.LaneConfig(4, 8, 1))
    A, B, C0, ldb = _operands(32, 64, 64, (4, 8, 1), True, seed=21)
    a = torch.from_numpy(A).to(dev)
    b = torch.from_numpy(B).to(dev)
    ctx.preprocess(a, b)
    c = torch.from_numpy(C0).to(dev)
    a.mul_(1.0)  # bumps the content version: stale
    with pytest.raises(mmm.StaleContextError):
        ctx.multiply(c, a, b)
    with pytest.raises(mmm.DimensionMismatchError):
        mmm.MmmContext(0, lane=mmm.LaneConfig(4, 8, 1)).preprocess(a, b[:10])
    bad = mmm.MmmContext(0, lane=mmm.LaneConfig(3, 8, 1))
    with pytest.raises(ValueError, match="group width 3 for f64"):
        bad.preprocess(a, b)
    f32ctx = mmm.MmmContext(0, lane=mmm.LaneConfig(4, 8, 1))
    with pytest.raises(ValueError, match="same dtype"):
        f32ctx.preprocess(a.float(), b)
