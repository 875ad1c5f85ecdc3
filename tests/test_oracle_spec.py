"""SPEC.md known answers and properties, asserted on the CPU oracle (the checker the GPU path
is compared against).  Each test names the SPEC line it encodes."""
import numpy as np
import pytest

from oracle import oracle as o


def test_code_examples():
    # SPEC.md:149-151 / :158-160
    rng = np.random.default_rng(0)
    c0 = rng.uniform(-1, 1, 64).astype(np.float32)
    b = rng.uniform(-1, 1, 64).astype(np.float32)
    assert np.array_equal(o.region_fma(0b00000000, c0.copy(), np.float32(0.5), b), c0)
    full = o.region_fma(0xFF, c0.copy(), np.float32(0.5), b)
    # 0.5*b is exact in fp32, so the fused and unfused results coincide
    assert np.array_equal(full, (np.float32(0.5) * b + c0).astype(np.float32))
    got = o.region_fma(0b01010000, c0.copy(), np.float32(0.5), b)
    changed = np.nonzero(got != c0)[0]
    assert set(changed) <= set(range(8, 16)) | set(range(24, 32))
    assert set(changed) == set(range(8, 16)) | set(range(24, 32))
    # code full, a = 1, c = 0 -> copy of b
    assert np.array_equal(o.region_fma(0xFF, np.zeros(64, np.float32), np.float32(1.0), b), b)


def test_kernel_exhaustive_vs_scalar():
    # acceptance 1: all 256 codes x random inputs; zero-bit lanes bit-exact, others fma
    rng = np.random.default_rng(1)
    for code in range(256):
        for _ in range(3):
            c0 = rng.uniform(-1, 1, 64).astype(np.float32)
            b = rng.uniform(-1, 1, 64).astype(np.float32)
            a = np.float32(rng.uniform(-1, 1))
            got = o.region_fma(code, c0.copy(), a, b)
            for j in range(8):
                sl = slice(8 * j, 8 * j + 8)
                if (code >> (7 - j)) & 1:
                    ref = (np.float64(a) * b[sl].astype(np.float64) + c0[sl]).astype(np.float32)
                    assert np.allclose(got[sl], ref, rtol=1e-6, atol=1e-7)
                else:
                    assert np.array_equal(got[sl].view(np.uint32), c0[sl].view(np.uint32))


def test_preprocess_b_examples():
    # SPEC.md:201-204
    B = np.zeros((4, 64), np.float32)
    assert (o.pattern_codes(B) == 0).all()
    B = np.ones((4, 128), np.float32)
    assert (o.pattern_codes(B) == 0xFF).all()
    B = np.zeros((1, 64), np.float32)
    B[0, 9] = 1.0
    B[0, 30] = -2.0
    assert o.pattern_codes(B)[0, 0] == 0b01010000


def test_preprocess_b_rescan_and_bplan_order():
    # SPEC.md:205, :224 (plan/rescan equivalence) and :188 (order)
    B = o.ref_generate(300, 500, "block_random", 0.6, 16, 5)
    codes = o.pattern_codes(B)
    K, nreg = codes.shape
    for k in range(0, K, 37):
        for r in range(nreg):
            want = 0
            for j in range(8):
                want = (want << 1) | int(np.any(B[k, r * 64 + 8 * j: r * 64 + 8 * j + 8] != 0))
            assert codes[k, r] == want
    plans = o.bplans(codes, leaf_dim=256)
    # 2 leaf rows x 2 leaf cols (nreg = 8 -> 4 regions per leaf)
    assert len(plans) == 4
    assert np.array_equal(plans[0], codes[:256, :4].ravel())
    assert np.array_equal(plans[1], codes[:256, 4:].ravel())
    assert np.array_equal(plans[3], codes[256:, 4:].ravel())
    assert sum(len(p) for p in plans) == codes.size


def test_preprocess_a_examples():
    # SPEC.md:211-213
    A = np.zeros((1, 16), np.float32)
    A[0, :8] = [5, 0, 0, 2, 0, 0, 0, 9]
    A[0, 8:] = 1.0
    counts, offsets = o.ablock_index(A, block_dim=256)
    assert counts.tolist() == [3, 8]
    assert offsets[0, :3].tolist() == [0, 3, 7] and (offsets[0, 3:] == 0xFF).all()
    assert (offsets[1] == 0xFF).all()  # full segment stores no offsets


def test_preprocess_a_roundtrip():
    # reconstruction from (counts, offsets) equals the non-zero set
    A = o.ref_generate(300, 520, "random", 0.7, 0, 9)
    K = 520
    counts, offsets = o.ablock_index(A, K=K, block_dim=256)
    rebuilt = np.zeros((300, K), bool)
    s = 0
    for bi in range(0, 300, 256):
        for bk in range(0, K, 256):
            for i in range(bi, min(bi + 256, 300)):
                for k0 in range(bk, min(bk + 256, K), 8):
                    n = counts[s]
                    offs = range(8) if n == 8 else offsets[s, :n]
                    for t in offs:
                        rebuilt[i, k0 + int(t)] = True
                    s += 1
    assert s == counts.size
    assert np.array_equal(rebuilt, A[:, :K] != 0)


def test_plan_stats_examples():
    # SPEC.md:218-221
    assert o.plan_stats(np.zeros((8, 4), np.uint32))[1] == 1.0
    assert o.plan_stats(np.full((8, 4), 255, np.uint32))[2] == 8.0
    B = o.ref_generate(1024, 1024, "block_random", 0.8, 64, 3)
    z = o.plan_stats(o.pattern_codes(B))[1]
    assert abs(z - 0.8) <= 0.01


def _pair(n, sa, sb, sb_struct="block_random", seed=1):
    A = o.ref_generate(n, n, "random", sa, 0, seed)
    B = o.ref_generate(n, n, sb_struct, sb, 0, seed + 100)
    return A, B


def test_multiply_counters_examples():
    # SPEC.md:282-283
    n = 256
    A = np.zeros((n, n), np.float32)
    B = o.ref_generate(n, n, "random", 0.0, 0, 1)
    C = np.zeros((n, n), np.float32)
    cnt = o.multiply_mmm(C, A, B)
    assert cnt["lane_fma_ops"] == 0 and not C.any()
    A = o.ref_generate(n, n, "random", 0.0, 0, 2)
    cnt = o.multiply_mmm(C, A, B)
    assert cnt["lane_fma_ops"] == n ** 3


@pytest.mark.parametrize("sa,sb", [(0.8, 0.8), (0.5, 0.25), (0.95, 0.5)])
def test_exact_work_identity_and_skip_identity(sa, sb):
    # SPEC.md:284, :297-298; acceptance 3
    A, B = _pair(256, sa, sb)
    C = np.zeros_like(A)
    cnt = o.multiply_mmm(C, A, B)
    assert cnt["lane_fma_ops"] == o.bruteforce_lane_ops(A, B)
    assert cnt["rows_skipped"] + int((A != 0).sum()) == A.size


def test_op_count_reduction():
    # acceptance 4: n = 2048 would be slow on CPU; the bound is scale-free, check at 1024
    A = o.ref_generate(1024, 1024, "random", 0.7, 0, 11)
    B = o.ref_generate(1024, 1024, "block_random", 0.7, 64, 12)
    assert o.bruteforce_lane_ops(A, B) <= 0.15 * 1024 ** 3


@pytest.mark.parametrize("struct", ["random", "block_random", "column", "block_column"])
@pytest.mark.parametrize("sa,sb", [(0.0, 0.0), (0.5, 0.8), (0.95, 0.25), (1.0, 0.5)])
def test_mmm_equals_simple(struct, sa, sb):
    # SPEC.md:296 grid (CPU slice): multiply_mmm == multiply_simple (bit-exact: skipped
    # terms are exact fma no-ops on finite data and C starts at +0)
    A = o.ref_generate(256, 256, "random", sa, 0, 3)
    B = o.ref_generate(256, 256, struct, sb, 0, 4)
    C1 = np.zeros_like(A)
    C2 = np.zeros_like(A)
    o.multiply_mmm(C1, A, B)
    o.multiply_simple(C2, A, B)
    assert np.array_equal(C1.view(np.uint32), C2.view(np.uint32))


def test_generator_statistics():
    # SPEC.md:104-105, acceptance 10
    for s in ["random", "block_random", "column", "block_column"]:
        m = o.ref_generate(1024, 1024, s, 0.8, 0, 42)
        assert abs((m == 0).mean() - 0.8) <= 0.01, s


def test_iid_generators():
    # BASELINE.json generators: i.i.d. element / block masks at the target rate
    a = o.gen_iid(1024, 1024, 5, mask_kind=1, p=0.8)
    assert abs((a == 0).mean() - 0.8) < 0.01
    assert a.min() >= -1 and a.max() <= 1
    b = o.gen_iid(1024, 1024, 6, mask_kind=2, p=0.8, block=16)
    blocks = (b.reshape(1024, 64, 16) != 0)
    assert (blocks.all(axis=2) | (~blocks).all(axis=2)).all()  # blocks all-zero or all-non-zero
    assert abs((~blocks.any(axis=2)).mean() - 0.8) < 0.01
    r = o.gen_iid(2048, 512, 7, value_kind=2, thresh=1.2815515655446004)
    assert abs((r == 0).mean() - 0.9) < 0.005
    g = o.gen_iid(1024, 512, 8, value_kind=1, sigma=0.02)
    assert abs(g.std() - 0.02) < 0.001
