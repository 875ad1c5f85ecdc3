"""GPU parity: the CUDA path through the C ABI against the CPU oracle on the same inputs.

Bar (BASELINE.json north_star): masks / index lists / codes / counters bit-exact; C within
|ΔC| <= 1e-5 * (|c0| + Σ|a||b|).  Two K2 paths are held to it:
  EXACT (K2-SIMT, forced with ALGO_SIMT_BCAST): replays the oracle's ascending-k fmaf chain,
        so C is bit-exact;
  AUTO  (the default): K1's cost model and guards pick K2-SIMT or K2-TC (fp16-split tcgen05
        MMAs, per-row / per-group power-of-two scales) on the device; checked against the
        tolerance, counters exact.
"""
import numpy as np
import pytest

from oracle import oracle as o

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2402_14118_b200 as mmm  # noqa: E402
from paper_2402_14118_b200 import _native as N  # noqa: E402
from paper_2402_14118_b200.api import MASK_BLOCK, MASK_ELEMENT, VALUE_NORMAL, VALUE_RELU  # noqa: E402

TOL = 1e-5  # north_star: relative to Σ_k |a_ik||b_kj|
EXACT = N.ALGO_SIMT_BCAST  # bit-exact K2-SIMT (device-side span choice)


@pytest.fixture(scope="module")
def ctx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return mmm.MmmContext(0)


def dev(x: np.ndarray):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def padded(x: np.ndarray, ld: int) -> np.ndarray:
    out = np.zeros((x.shape[0], ld), dtype=np.float32)
    out[:, : x.shape[1]] = x
    return out


def run_gpu(ctx, A, B, C0=None, algo=N.ALGO_AUTO, N_=None):
    """A: M x lda (logical K = B rows), B: K x ldb (logical N_), C0: M x ldb."""
    M = A.shape[0]
    K = B.shape[0]
    N_ = B.shape[1] if N_ is None else N_
    a = dev(A)[:, :K] if K != A.shape[1] else dev(A)
    b = dev(B)[:, :N_] if N_ != B.shape[1] else dev(B)
    cfull = dev(np.zeros((M, B.shape[1]), np.float32) if C0 is None else C0)
    c = cfull[:, :N_] if N_ != B.shape[1] else cfull
    ctx.set_algo(algo)
    ctx.preprocess(a, b)
    cnt = mmm.multiply_mmm(ctx, c, a, b)
    torch.cuda.synchronize()
    ctx.set_algo(N.ALGO_AUTO)
    return cfull.cpu().numpy(), cnt


def run_oracle(A, B, C0=None):
    C = np.zeros((A.shape[0], B.shape[1]), np.float32) if C0 is None else C0.copy()
    Aq = np.ascontiguousarray(A[:, : B.shape[0]])
    cnt = o.multiply_mmm(C, Aq, B)
    return C, cnt


def assert_counters(cnt, ocnt):
    assert cnt.lane_fma_ops == ocnt["lane_fma_ops"]
    assert cnt.kernel_invocations == ocnt["kernel_invocations"]
    assert cnt.rows_skipped == ocnt["rows_skipped"]
    assert cnt.regions_skipped_by_zero_code == ocnt["regions_skipped_by_zero_code"]


def within_tol(C, Cr, A, B, C0=None):
    """|C - Cr| <= TOL * (|c0| + Σ|a||b|), fp64 denominators."""
    K = B.shape[0]
    Aq = np.ascontiguousarray(A[:, :K])
    if C0 is None:
        bad, worst = o.check_tolerance(C, Cr, Aq, B, tol=TOL)
        return bad == 0, worst
    den = np.abs(Aq).astype(np.float64) @ np.abs(B).astype(np.float64) + np.abs(C0).astype(np.float64)
    err = np.abs(C.astype(np.float64) - Cr.astype(np.float64))
    ok = err <= TOL * den
    worst = float(np.max(np.where(den > 0, err / np.where(den > 0, den, 1), 0)))
    return bool(ok.all()), worst


def check_auto(ctx, A, B, Cr, ocnt, C0=None, N_=None):
    """The default (AUTO) path: tolerance, exact counters, padding zero; returns the path taken."""
    C, cnt = run_gpu(ctx, A, B, C0=C0, algo=N.ALGO_AUTO, N_=N_)
    ok, worst = within_tol(C, Cr, A, B, C0=C0)
    assert ok, worst
    assert worst < 0.5 * TOL, worst
    assert_counters(cnt, ocnt)
    if N_ is not None:
        assert (C[:, N_:] == 0).all()
    return ctx.last_algo()


def bitexact(x, y):
    return np.array_equal(np.ascontiguousarray(x).view(np.uint32), np.ascontiguousarray(y).view(np.uint32))


def gen_pair(seed, M, K, N_, zA, zB, bw, a_kind=0, b_kind=0, a_thresh=0.0, b_sigma=1.0):
    A = o.gen_iid(M, K, mmm.matrix_seed(seed, "A"), value_kind=a_kind, thresh=a_thresh, mask_kind=1 if zA else 0,
                  p=zA, ld=mmm.round_up(K, 64))  # Matrix layout: padded, zero padding
    ldb = mmm.round_up(N_, 64)
    B = o.gen_iid(K, N_, mmm.matrix_seed(seed, "B"), value_kind=b_kind, sigma=b_sigma, mask_kind=2 if zB else 0,
                  p=zB, block=bw, ld=ldb)
    return A, B


# ------------------------------------------------------------------------------ K1
@pytest.mark.parametrize("M,K,N_", [(1024, 1024, 1024), (100, 77, 130), (33, 300, 64), (257, 1000, 600)])
def test_k1_masks_codes_csr_bitexact(ctx, M, K, N_):
    A, B = gen_pair(11, M, K, N_, 0.8, 0.8, 16)
    a, b = dev(A)[:, :K], dev(B)[:, :N_]
    ctx.preprocess(a, b)
    ldb = B.shape[1]
    assert np.array_equal(ctx.export_b_codes(K, ldb), o.pattern_codes(B).astype(np.uint8))
    assert np.array_equal(ctx.export_a_bitmap(M, K), o.a_bitmap(A, K=K))
    rp, cols = ctx.export_a_csr(M)
    orp, ocols = o.a_csr(A, K=K)
    assert np.array_equal(rp, orp) and np.array_equal(cols, ocols)
    idx = ctx.export_ablock_index(M, K, 256)
    oc, oo = o.ablock_index(A, K=K, block_dim=256)
    assert np.array_equal(idx.counts, oc) and np.array_equal(idx.offsets, oo)
    plans = ctx.export_bplans(K, ldb, 256)
    oplans = o.bplans(o.pattern_codes(B), leaf_dim=256)
    assert len(plans) == len(oplans)
    for p, q in zip(plans, oplans):
        assert np.array_equal(p.codes, q.astype(np.uint8))
    st = ctx.plan_stats()
    n, z, mp = o.plan_stats(o.pattern_codes(B))
    assert st.region_count == n and st.zero_region_fraction == pytest.approx(z, abs=0) and st.mean_popcount == \
        pytest.approx(mp, abs=0)


def test_k1_zero_semantics(ctx):
    # ±0 are zero; NaN, denormals, inf are non-zero (matrix.hpp:152/174)
    A = np.zeros((32, 64), np.float32)
    A[0, 0] = -0.0
    A[0, 1] = np.float32(1e-45)  # denormal
    A[0, 2] = np.nan
    A[0, 3] = np.inf
    B = np.zeros((64, 64), np.float32)
    B[0, 8] = np.float32(1e-45)
    B[1, 0] = -0.0
    ctx.preprocess(dev(A), dev(B))
    bits = ctx.export_a_bitmap(32, 64)
    assert bits[0, 0] == 0b1110
    codes = ctx.export_b_codes(64, 64)
    assert codes[0, 0] == 0b01000000 and codes[1, 0] == 0


# ------------------------------------------------------------------------------ K2
@pytest.mark.parametrize("algo", [EXACT, N.ALGO_SIMT_SPAN8, N.ALGO_SIMT_SPAN16])
def test_cfg1_bitexact(ctx, algo):
    # BASELINE configs[0]: 1024^3, A 0.8 element zeros, B 16-wide blocks 0.8 zeros
    A, B = gen_pair(1, 1024, 1024, 1024, 0.8, 0.8, 16)
    C, cnt = run_gpu(ctx, A, B, algo=algo)
    Cr, ocnt = run_oracle(A, B)
    assert bitexact(C, Cr)
    assert_counters(cnt, ocnt)


def test_cfg1_auto(ctx):
    A, B = gen_pair(1, 1024, 1024, 1024, 0.8, 0.8, 16)
    Cr, ocnt = run_oracle(A, B)
    check_auto(ctx, A, B, Cr, ocnt)


@pytest.mark.parametrize("struct", ["random", "block_random", "column", "block_column"])
@pytest.mark.parametrize("sa", [0.0, 0.25, 0.5, 0.8, 0.95, 1.0])
@pytest.mark.parametrize("n", [256, 512])
def test_spec_grid_bitexact(ctx, struct, sa, n):
    # SPEC.md:296 / acceptance 2 grid (sizes 256/512 here; 1024 in the slow set)
    for sb in (0.0, 0.5, 0.95):
        A = o.ref_generate(n, n, "random", sa, 0, 3)
        B = o.ref_generate(n, n, struct, sb, 0, 4)
        C, cnt = run_gpu(ctx, A, B, algo=EXACT)
        Cr, ocnt = run_oracle(A, B)
        assert bitexact(C, Cr), (struct, sa, sb)
        assert_counters(cnt, ocnt)
        check_auto(ctx, A, B, Cr, ocnt)


@pytest.mark.parametrize("M,K,N_", [(100, 77, 130), (33, 300, 64), (257, 1000, 600), (1, 5, 1), (129, 65, 257)])
def test_ragged_shapes_and_accumulate(ctx, M, K, N_):
    # edge tiles in every dimension, K not a multiple of 4/32, N padded to 64; C += A*B
    A, B = gen_pair(5, M, K, N_, 0.6, 0.6, 8)
    rng = np.random.default_rng(M)
    C0 = np.zeros((M, B.shape[1]), np.float32)
    C0[:, :N_] = rng.uniform(-1, 1, (M, N_)).astype(np.float32)
    C, cnt = run_gpu(ctx, A, B, C0=C0, N_=N_, algo=EXACT)
    Cr, ocnt = run_oracle(A, B, C0=C0)
    assert bitexact(C, Cr)
    assert (C[:, N_:] == 0).all()  # padding stays zero
    assert_counters(cnt, ocnt)
    check_auto(ctx, A, B, Cr, ocnt, C0=C0, N_=N_)


@pytest.mark.parametrize("zA,zB,bw", [(0.6, 0.6, 8), (0.7, 0.95, 16), (0.8, 0.8, 32), (0.95, 0.6, 16),
                                      (0.9, 0.9, 8)])
def test_cfg2_cells_bitexact(ctx, zA, zB, bw):
    # BASELINE configs[1] cells at the full 4096^3 size
    A, B = gen_pair(2, 4096, 4096, 4096, zA, zB, bw)
    C, cnt = run_gpu(ctx, A, B, algo=EXACT)
    Cr, ocnt = run_oracle(A, B)
    assert bitexact(C, Cr)
    assert_counters(cnt, ocnt)
    check_auto(ctx, A, B, Cr, ocnt)


def test_cfg3_mlp_down_projection(ctx):
    # BASELINE configs[2]: A = ReLU(G - t) 2048x16384 (~90% zeros), B ~ N(0, 0.02) with
    # 32-wide blocks kept w.p. 0.1
    A, B = gen_pair(3, 2048, 16384, 4096, 0.0, 0.9, 32, a_kind=VALUE_RELU, a_thresh=1.2815515655446004,
                    b_kind=VALUE_NORMAL, b_sigma=0.02)
    assert abs((A == 0).mean() - 0.9) < 0.01
    C, cnt = run_gpu(ctx, A, B, algo=EXACT)
    Cr, ocnt = run_oracle(A, B)
    assert bitexact(C, Cr)
    assert_counters(cnt, ocnt)
    check_auto(ctx, A, B, Cr, ocnt)


def test_cfg4_skinny_decode(ctx):
    # BASELINE configs[3]: 64 x 12288 x 49152, A ReLU ~95% zeros, B 16-wide blocks kept 0.15
    A, B = gen_pair(4, 64, 12288, 49152, 0.0, 0.85, 16, a_kind=VALUE_RELU, a_thresh=1.6448536269514722,
                    b_kind=VALUE_NORMAL, b_sigma=0.02)
    C, cnt = run_gpu(ctx, A, B, algo=EXACT)
    Cr, ocnt = run_oracle(A, B)
    assert bitexact(C, Cr)
    assert_counters(cnt, ocnt)
    check_auto(ctx, A, B, Cr, ocnt)
    # forced K2-TC on the skinny shape: one 128-row tile, so the CTA pair's second row tile
    # is all padding; fp16 scales from ReLU / N(0, 0.02) operands
    for algo in (N.ALGO_TC, N.ALGO_TC32):
        C, cnt = run_gpu(ctx, A, B, algo=algo)
        ok, worst = within_tol(C, Cr, A, B)
        assert ok and worst < 0.5 * TOL, (algo, worst)
        assert_counters(cnt, ocnt)


def test_cfg5_row_shards(ctx):
    # BASELINE configs[4]: 32768 x 8192 x 8192 at 0.85/0.85; each shard of a 2/4/8-way
    # row partition is multiplied on its own (the per-rank work of the sharded run) and
    # sampled rows of every shard are compared with the oracle.
    M, K, N_ = 32768, 8192, 8192
    A, B = gen_pair(5, M, K, N_, 0.85, 0.85, 16)
    b = dev(B)
    rng = np.random.default_rng(5)
    for world in (2, 4, 8):
        for rank in range(world):
            r0, r1 = mmm.shard_rows(M, world, rank)
            a = dev(A[r0:r1])
            rows = np.sort(rng.choice(r1 - r0, 8, replace=False))
            Cr = np.zeros((8, N_), np.float32)
            Ar = np.ascontiguousarray(A[r0:r1][rows][:, :K])
            o.multiply_mmm(Cr, Ar, B)
            for algo in (EXACT, N.ALGO_AUTO):
                c = torch.zeros((r1 - r0, N_), dtype=torch.float32, device="cuda")
                ctx.set_algo(algo)
                ctx.preprocess(a, b)
                mmm.multiply_mmm(ctx, c, a, b)
                Cg = c.cpu().numpy()[rows]
                if algo == EXACT:
                    assert bitexact(Cg, Cr), (world, rank)
                else:
                    bad, worst = o.check_tolerance(Cg, Cr, Ar, B, tol=TOL)
                    assert bad == 0, (world, rank, worst)
            ctx.set_algo(N.ALGO_AUTO)


# ------------------------------------------------------------------- other entry points
def test_multiply_simple_bitexact(ctx):
    A, B = gen_pair(9, 300, 200, 256, 0.5, 0.5, 8)
    C = torch.zeros((300, 256), dtype=torch.float32, device="cuda")
    mmm.multiply_simple(C, dev(A)[:, :200], dev(B), ctx=ctx)
    Cr = np.zeros((300, 256), np.float32)
    o.multiply_simple(Cr, np.ascontiguousarray(A[:, :200]), B)
    assert bitexact(C.cpu().numpy(), Cr)


def test_dense_algo_matches(ctx):
    A, B = gen_pair(10, 256, 256, 256, 0.8, 0.8, 16)
    C, cnt = run_gpu(ctx, A, B, algo=N.ALGO_DENSE)
    Cr, ocnt = run_oracle(A, B)
    assert bitexact(C, Cr)
    assert_counters(cnt, ocnt)


def test_multiply_host_path(ctx):
    A, B = gen_pair(12, 200, 320, 192, 0.8, 0.8, 16)
    Cr, ocnt = run_oracle(A, B)
    for algo in (EXACT, N.ALGO_AUTO):
        ctx.set_algo(algo)
        C = np.zeros((200, 192), np.float32)
        cnt = mmm.multiply_host(C, A, B, ctx=ctx)
        if algo == EXACT:
            assert bitexact(C, Cr)
        else:
            ok, worst = within_tol(C, Cr, A, B)
            assert ok, worst
        assert_counters(cnt, ocnt)
    ctx.set_algo(N.ALGO_AUTO)


def test_auto_choice_and_switch(ctx):
    # a dense cell goes to K2-TC; forcing the other path on an AUTO plan re-packs its
    # operands (both stay correct); a very sparse, short cell is correct either way
    A, B = gen_pair(15, 2048, 2048, 2048, 0.6, 0.6, 8)
    Cr, ocnt = run_oracle(A, B)
    assert check_auto(ctx, A, B, Cr, ocnt) == N.ALGO_TC
    a, b = dev(A), dev(B)
    ctx.set_algo(N.ALGO_AUTO)
    ctx.preprocess(a, b)
    ctx.set_algo(EXACT)  # plan built for AUTO (TC chosen, SIMT rows gated out)
    c = torch.zeros((2048, 2048), dtype=torch.float32, device="cuda")
    mmm.multiply_mmm(ctx, c, a, b)
    assert bitexact(c.cpu().numpy(), Cr)
    ctx.set_algo(N.ALGO_AUTO)
    A2, B2 = gen_pair(16, 128, 4096, 4096, 0.99, 0.99, 8)
    Cr2, ocnt2 = run_oracle(A2, B2)
    assert check_auto(ctx, A2, B2, Cr2, ocnt2) in (N.ALGO_TC, N.ALGO_SIMT_SPAN8, N.ALGO_SIMT_SPAN16)


def test_stale_and_errors(ctx):
    A, B = gen_pair(13, 128, 128, 128, 0.8, 0.8, 16)
    a, b = dev(A), dev(B)
    c = torch.zeros((128, 128), dtype=torch.float32, device="cuda")
    ctx.preprocess(a, b)
    a.add_(0.0)  # in-place write bumps the version: the plan is stale
    with pytest.raises(mmm.StaleContextError):
        mmm.multiply_mmm(ctx, c, a, b)
    ctx.preprocess(a, b)
    with pytest.raises(ValueError):
        mmm.multiply_parallel(ctx, c, a, b, 0)
    cnt1 = mmm.multiply_parallel(ctx, c, a, b, 8)
    assert cnt1.lane_fma_ops == ctx.planned_counters().lane_fma_ops
    other = mmm.MmmContext(0, lane=mmm.LaneConfig(4, 8, 1))
    other.preprocess(a, b)  # a non-default lane runs the lane-general kernels (tests/test_gpu_lanes.py)
    with pytest.raises(mmm.DimensionMismatchError):
        ctx.preprocess(a, dev(np.zeros((64, 128), np.float32)))
    with pytest.raises(ValueError):  # mixed dtypes
        ctx.preprocess(a.double(), b)
    with pytest.raises(mmm.UnsupportedError):  # no GPU kernel for half precision
        ctx.preprocess(a.half(), b.half())


def test_split_preprocess_paths(ctx):
    # preprocess_b / preprocess_a on their own: the K1 scratch of only one
    # operand is re-zeroed, the gated packs re-run on the device choice, and the plans follow
    # the new operand (AUTO, K2-TC for these densities; the exact path beside it)
    M, K, N_ = 512, 768, 640
    A, B = gen_pair(31, M, K, N_, 0.6, 0.7, 16)
    A2, B2 = gen_pair(32, M, K, N_, 0.7, 0.6, 8)
    a, b, a2, b2 = dev(A), dev(B), dev(A2), dev(B2)
    for algo in (N.ALGO_AUTO, EXACT):
        ctx.set_algo(algo)
        ctx.preprocess(a, b)
        for which, aa, bb, An, Bn in (("b", a, b2, A, B2), ("a", a2, b2, A2, B2)):
            if which == "b":
                ctx.preprocess_b_only(bb)
            else:
                ctx.preprocess_a_only(aa)
            c = torch.zeros((M, N_), dtype=torch.float32, device="cuda")
            cnt = mmm.multiply_mmm(ctx, c, aa, bb)
            Cr, ocnt = run_oracle(An, Bn)
            if algo == EXACT:
                assert bitexact(c.cpu().numpy(), Cr), which
            else:
                ok, worst = within_tol(c.cpu().numpy(), Cr, An, Bn)
                assert ok and worst < 0.5 * TOL, (which, worst)
            assert_counters(cnt, ocnt)
    ctx.set_algo(N.ALGO_AUTO)


def test_parallel_determinism(ctx):
    # identical bits and counters across runs and worker counts
    A, B = gen_pair(14, 512, 512, 512, 0.8, 0.8, 16)
    outs = []
    for w in (1, 4, 8):
        a, b = dev(A), dev(B)
        c = torch.zeros((512, 512), dtype=torch.float32, device="cuda")
        ctx.preprocess(a, b)
        cnt = mmm.multiply_parallel(ctx, c, a, b, w)
        outs.append((c.cpu().numpy(), cnt))
    for c, cnt in outs[1:]:
        assert bitexact(c, outs[0][0]) and cnt == outs[0][1]


def test_device_generator_matches_oracle(ctx):
    # uniform values and both mask kinds are bit-identical to the oracle's host generator
    for kw in (dict(mask_kind=MASK_ELEMENT, p=0.8), dict(mask_kind=MASK_BLOCK, p=0.7, block=16), dict()):
        t = torch.empty((257, 320), dtype=torch.float32, device="cuda")
        mmm.generate(t, seed=1234, cols=300, ctx=ctx, **kw)
        host = o.gen_iid(257, 300, 1234, ld=320, **kw)
        assert bitexact(t.cpu().numpy(), host)
    # normal modes: same formula through device log1p/cos; allow rare last-ulp differences
    t = torch.empty((512, 512), dtype=torch.float32, device="cuda")
    mmm.generate(t, seed=99, value_kind=VALUE_RELU, thresh=1.2815515655446004, ctx=ctx)
    host = o.gen_iid(512, 512, 99, value_kind=VALUE_RELU, thresh=1.2815515655446004)
    g = t.cpu().numpy()
    assert ((g == 0) == (host == 0)).mean() > 0.9999
    assert np.allclose(g, host, rtol=1e-6, atol=1e-7)


# --------------------------------------------------------------- K2-TC (tcgen05 3xTF32)
@pytest.mark.parametrize("M,K,N_,zA,zB,bw", [(1024, 1024, 1024, 0.8, 0.8, 16), (100, 77, 130, 0.6, 0.6, 8),
                                            (257, 1000, 600, 0.0, 0.0, 16), (4096, 4096, 4096, 0.6, 0.6, 32),
                                            (4096, 4096, 4096, 0.95, 0.95, 8), (129, 65, 257, 1.0, 0.5, 16)])
@pytest.mark.parametrize("algo", [N.ALGO_TC, N.ALGO_TC32])
def test_tc_tolerance(ctx, M, K, N_, zA, zB, bw, algo):
    # north_star: |C_gpu - C_ref| <= 1e-5 * Σ_k |a_ik||b_kj| (fp64 denominator); exact counters
    # (ALGO_TC: fp16 split with power-of-two operand scales; ALGO_TC32: 3xTF32)
    A, B = gen_pair(21, M, K, N_, zA, zB, bw)
    C, cnt = run_gpu(ctx, A, B, algo=algo, N_=N_)
    Cr, ocnt = run_oracle(A, B)
    bad, worst = o.check_tolerance(C, Cr, np.ascontiguousarray(A[:, :K]), B, tol=TOL)
    assert bad == 0, worst
    assert worst < 0.5 * TOL  # margin: typical worst ~4e-6 at dA = dB = 0.4
    assert (C[:, N_:] == 0).all()
    assert_counters(cnt, ocnt)


@pytest.mark.parametrize("sa,sb", [(1e6, 1e-8), (3e-20, 2e15), (65504.0, 65504.0), (1.0, 0.02)])
def test_tc_f16_scaled_operands(ctx, sa, sb):
    # the fp16 split scales each operand by a power of two (max|x| -> [2^14, 2^15)): operands
    # far outside fp16's range stay within the tolerance
    M, K, N_ = 384, 1024, 384
    A, B = gen_pair(23, M, K, N_, 0.6, 0.7, 16)
    A = (A * np.float32(sa)).astype(np.float32)
    B = (B * np.float32(sb)).astype(np.float32)
    C, cnt = run_gpu(ctx, A, B, algo=N.ALGO_TC, N_=N_)
    Cr, ocnt = run_oracle(A, B)
    bad, worst = o.check_tolerance(C, Cr, np.ascontiguousarray(A[:, :K]), B, tol=TOL)
    assert bad == 0, worst
    assert worst < 0.5 * TOL, worst
    assert_counters(cnt, ocnt)


def test_auto_range_guard(ctx):
    # an operand maximum outside the fp16 split's scale range (max exponent > 114) keeps AUTO on the
    # exact K2-SIMT path
    A, B = gen_pair(24, 512, 512, 512, 0.6, 0.6, 16)
    A = (A * np.float32(2.0 ** 116)).astype(np.float32)  # max|A| in [2^115, 2^116)
    Cr, ocnt = run_oracle(A, B)
    C, cnt = run_gpu(ctx, A, B, algo=N.ALGO_AUTO)
    assert ctx.last_algo() in (N.ALGO_SIMT_SPAN8, N.ALGO_SIMT_SPAN16)
    assert bitexact(C, Cr)
    assert_counters(cnt, ocnt)


def test_tc_accumulate(ctx):
    # c += a*b into a non-zero C: the TC path adds its fp32 product to C once, so the
    # tolerance extends to Σ|a||b| + |c0| (the rounding of the final add is relative to c0)
    M, K, N_ = 300, 520, 320
    A, B = gen_pair(22, M, K, N_, 0.8, 0.8, 16)
    C0 = np.random.default_rng(3).uniform(-1, 1, (M, B.shape[1])).astype(np.float32)
    C0[:, N_:] = 0
    C, _ = run_gpu(ctx, A, B, C0=C0, algo=N.ALGO_TC, N_=N_)
    Cr, _ = run_oracle(A, B, C0=C0)
    den = np.abs(A[:, :K]).astype(np.float64) @ np.abs(B).astype(np.float64) + np.abs(C0).astype(np.float64)
    assert (np.abs(C.astype(np.float64) - Cr) <= TOL * den).all()


def test_cpp_dropin(ctx):
    # the reference-side C++ caller (SPEC engine API on the reference's Matrix<float>) linked
    # against libmmmcu.so through include/mmm_cuda.hpp
    import os
    import subprocess

    exe = os.path.join(os.path.dirname(N.LIB_PATH), "dropin_test")
    if not os.path.exists(exe):
        pytest.skip("dropin_test not built (needs the reference headers at build time)")
    out = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "DROPIN OK" in out.stdout


def test_nonfinite_operands_stay_exact(ctx):
    # Inf / NaN are non-zero (matrix.hpp:152/174) and propagate through the reference's fmaf
    # chain; K2-TC would form 0 * Inf terms the reference never forms, so K1 flags
    # non-finite operands and AUTO keeps the exact K2-SIMT path
    A, B = gen_pair(17, 512, 512, 512, 0.6, 0.6, 8)
    A[3, 5] = np.inf
    A[10, 20] = -np.inf
    B[7, 9] = np.nan
    B[30, 100] = np.inf
    Cr, ocnt = run_oracle(A, B)
    C, cnt = run_gpu(ctx, A, B, algo=N.ALGO_AUTO)
    assert ctx.last_algo() in (N.ALGO_SIMT_SPAN8, N.ALGO_SIMT_SPAN16)
    assert (np.isnan(C) == np.isnan(Cr)).all()
    fin = ~np.isnan(Cr)
    assert bitexact(C[fin], Cr[fin])
    assert np.isinf(Cr).any() and np.isnan(Cr).any()
    assert_counters(cnt, ocnt)


def test_subnormal_operands_stay_exact(ctx):
    # subnormals are non-zero (matrix.hpp:174); tf32 tensor-core operands would flush them,
    # so AUTO keeps K2-SIMT (bit-exact) when K1 sees one
    A, B = gen_pair(18, 256, 256, 256, 0.6, 0.6, 8)
    A[:, 7] = np.float32(1e-40)  # a whole column of subnormals
    Cr, ocnt = run_oracle(A, B)
    C, cnt = run_gpu(ctx, A, B, algo=N.ALGO_AUTO)
    assert ctx.last_algo() in (N.ALGO_SIMT_SPAN8, N.ALGO_SIMT_SPAN16)
    assert bitexact(C, Cr)
    assert_counters(cnt, ocnt)
