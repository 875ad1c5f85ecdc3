"""Pin the CPU oracle (oracle/mmm_oracle.c) to the reference's OWN compiled code through the
fixtures of tests/golden/gen_golden.py (no /root/reference needed at run time)."""
import numpy as np
import pytest

from oracle import oracle as o

INV = {v: k for k, v in o.STRUCTURES.items()}


def test_generators_match_reference(golden):
    # generate<float> (matgen.hpp:77-148) restated in C: bit-identical for every structure
    for t in range(int(golden["gen_n"][0])):
        s, r, c, bl, seed = (int(x) for x in golden[f"gen{t}_meta"])
        tgt = float(golden[f"gen{t}_target"][0])
        got = o.ref_generate(r, c, INV[s], tgt, bl, seed)
        want = golden[f"gen{t}"]
        assert got.shape == want.shape
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), (INV[s], tgt, bl, seed)


@pytest.mark.parametrize("p", [8, 4, 12, 16])
def test_region_fma_matches_kernel_table(golden, p):
    # KernelTable<float>::apply (kernel_table.hpp:50-54): MSB-first groups, fused fma
    codes = golden[f"kt{p}_codes"]
    c0, b, a = golden[f"kt{p}_c0"], golden[f"kt{p}_b"], float(golden[f"kt{p}_a"][0])
    for code, want in zip(codes, golden[f"kt{p}_out"]):
        got = o.region_fma(int(code), c0.copy(), np.float32(a), b, group_width=8, pattern_bits=p)
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), (p, int(code))


def test_kernel_table_build_errors(golden):
    # reference: invalid_argument (status 1) for p outside [1,16] and unsupported G
    assert list(golden["kt_bad_status"]) == [1] * len(golden["kt_bad"])


def test_multiply_matches_reference_kernel_table(golden):
    # the SPEC multiply over the reference's compiled kernels == the oracle's multiply_mmm
    A, B, Cw = golden["mm_A"], golden["mm_B"], golden["mm_C"]
    C = np.zeros_like(Cw)
    cnt = o.multiply_mmm(C, A, B)
    assert np.array_equal(C.view(np.uint32), Cw.view(np.uint32))
    want = [int(x) for x in golden["mm_counters"]]
    assert [cnt["kernel_invocations"], cnt["lane_fma_ops"], cnt["rows_skipped"],
            cnt["regions_skipped_by_zero_code"]] == want


def test_mmmb_header(golden):
    # MMMB format (matrix_io.hpp:11-13): magic, version 1, dtype 0, rows, cols, payload
    raw = golden["mmmb_eye4"].tobytes()
    assert raw[:4] == b"MMMB"
    assert np.frombuffer(raw[4:12], dtype=np.uint32).tolist() == [1, 0]
    assert np.frombuffer(raw[12:28], dtype=np.uint64).tolist() == [4, 4]
    payload = np.frombuffer(raw[28:], dtype=np.float32).reshape(4, 4)
    assert np.array_equal(payload, np.eye(4, dtype=np.float32) * np.float32(1.5))


LANES32 = [(1, 8, 1), (2, 8, 1), (4, 8, 1), (4, 4, 4), (8, 2, 4), (32, 8, 2), (2, 16, 2)]
LANES64 = [(4, 8, 1), (2, 16, 1), (8, 8, 1)]


@pytest.mark.parametrize("lane", LANES32)
def test_region_fma_other_lanes(golden, lane):
    # KernelTable<float> for every compiled group width (kernel_table.cpp:47-57) and P != 8
    w, p, v = lane
    tag = f"ktl_{w}_{p}_{v}"
    c0, b, a = golden[tag + "_c0"], golden[tag + "_b"], float(golden[tag + "_a"][0])
    for code, want in zip(golden[tag + "_codes"], golden[tag + "_out"]):
        got = o.region_fma(int(code), c0.copy(), np.float32(a), b, group_width=w * v, pattern_bits=p)
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), (lane, int(code))


@pytest.mark.parametrize("lane", LANES64)
def test_region_fma_f64(golden, lane):
    # KernelTable<double> (kernel_table.cpp:94-95): fma per element of each set group
    w, p, v = lane
    tag = f"kt64_{w}_{p}_{v}"
    c0, b, a = golden[tag + "_c0"], golden[tag + "_b"], float(golden[tag + "_a"][0])
    for code, want in zip(golden[tag + "_codes"], golden[tag + "_out"]):
        got = o.region_fma(int(code), c0.copy(), a, b, group_width=w * v, pattern_bits=p)
        assert got.dtype == np.float64
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), (lane, int(code))


def test_multiply_other_lanes_and_f64(golden):
    # the SPEC multiply over the reference's KernelTable<T> for non-default lanes and f64
    for t in range(int(golden["mml_n"][0])):
        f64, w, p, v, M, K, N = (int(x) for x in golden[f"mml{t}_meta"])
        A, B, C0, want = (golden[f"mml{t}_{x}"] for x in ("A", "B", "C0", "C"))
        C = C0.copy()
        cnt = o.multiply_mmm(C, A, B, K=K, N=B.shape[1], group_width=w * v, pattern_bits=p)
        view = np.uint64 if f64 else np.uint32
        assert C.dtype == want.dtype
        assert np.array_equal(C.view(view), want.view(view)), t
        assert [cnt["kernel_invocations"], cnt["lane_fma_ops"], cnt["rows_skipped"],
                cnt["regions_skipped_by_zero_code"]] == [int(x) for x in golden[f"mml{t}_counters"]], t
