"""Generate the golden fixtures from the REFERENCE ITSELF (compiled from /root/reference by
oracle/Makefile into oracle/_ref/libmmmref.so).  Run in the build container only:

    make -C oracle ref && python tests/golden/gen_golden.py

The reference ships no tests or golden vectors, so these fixtures are what
pins the oracle's restatement (tests/test_oracle_golden.py) to the reference's own code:
  * generate<float> (matgen.hpp:77-148) for all four structures, several seeds/targets;
  * KernelTable<float>::build/apply (kernel_table.cpp:64-92, kernel_table.hpp:50-54) for
    every code at P=8 and sampled codes at P=4/12/16, and the build errors;
  * the SPEC multiply_parallel over the reference kernel table (ref_driver.cpp) on a small
    case: C and WorkCounters;
  * an MMMB file written by the reference writer (matrix_io.cpp:59-71).
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle as o  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def main():
    fx = {}
    # ---- generators
    cases = [
        ("random", 0.8, 0, 42, 37, 100),
        ("random", 0.25, 0, 7, 64, 64),
        ("block_random", 0.8, 0, 42, 40, 256),
        ("block_random", 0.7, 16, 3, 33, 130),
        ("column", 0.5, 0, 7, 20, 96),
        ("block_column", 0.6, 0, 11, 24, 200),
        ("block_column", 0.9, 16, 5, 24, 128),
    ]
    for t, (s, tgt, bl, seed, r, c) in enumerate(cases):
        fx[f"gen{t}_meta"] = np.array([o.STRUCTURES[s], r, c, bl, seed], dtype=np.int64)
        fx[f"gen{t}_target"] = np.array([tgt])
        fx[f"gen{t}"] = o.ref_generate_compiled(r, c, s, tgt, bl, seed)
    fx["gen_n"] = np.array([len(cases)])

    # ---- kernel table
    rng = np.random.default_rng(20240220)
    for p in (8, 4, 12, 16):
        R = 8 * p
        n_codes = 1 << p
        codes = np.arange(n_codes) if p <= 8 else np.unique(
            np.concatenate([[0, n_codes - 1], rng.integers(0, n_codes, 300)]))
        c0 = rng.uniform(-2, 2, R).astype(np.float32)
        b = rng.uniform(-2, 2, R).astype(np.float32)
        a = np.float32(rng.uniform(-2, 2))
        outs = []
        for code in codes:
            st, c = o.ref_kernel_apply(int(code), c0, a, b, lane=(8, p, 1))
            assert st == 0
            outs.append(c)
        fx[f"kt{p}_codes"] = codes.astype(np.uint32)
        fx[f"kt{p}_c0"] = c0
        fx[f"kt{p}_b"] = b
        fx[f"kt{p}_a"] = np.array([a], dtype=np.float32)
        fx[f"kt{p}_out"] = np.stack(outs)
    # build errors (kernel_table.cpp:66-72): (w, p, v) -> status (1 = invalid_argument)
    bad = [(8, 0, 1), (8, 17, 1), (3, 8, 1), (8, 8, 3), (128, 8, 1)]
    fx["kt_bad"] = np.array(bad, dtype=np.int64)
    fx["kt_bad_status"] = np.array(
        [o.ref_kernel_apply(0, np.zeros(max(8 * max(p, 1) * w * v, 8), np.float32), 1.0,
                            np.zeros(max(8 * max(p, 1) * w * v, 8), np.float32), lane=(w, p, v))[0]
         for (w, p, v) in bad], dtype=np.int64)

    # ---- SPEC multiply over the reference kernel table (small)
    A = o.ref_generate_compiled(96, 192, "random", 0.8, 0, 101)
    B = o.ref_generate_compiled(192, 160, "block_random", 0.8, 16, 202)
    Aq = np.ascontiguousarray(A[:, :192])
    C = np.zeros((96, B.shape[1]), dtype=np.float32)
    cnt = o.ref_multiply_parallel(C, Aq, B)
    fx["mm_A"] = Aq
    fx["mm_B"] = B
    fx["mm_C"] = C
    fx["mm_counters"] = np.array([cnt["kernel_invocations"], cnt["lane_fma_ops"], cnt["rows_skipped"],
                                  cnt["regions_skipped_by_zero_code"]], dtype=np.uint64)

    # ---- other lanes and f64: KernelTable<float> for every compiled
    # group width, KernelTable<double> at the f64 default lane, and the SPEC multiply over
    # them (ref_driver.cpp multiply_lane) on small cases
    for (w, p, v) in ((1, 8, 1), (2, 8, 1), (4, 8, 1), (4, 4, 4), (8, 2, 4), (32, 8, 2), (2, 16, 2)):
        G, R = w * v, w * p * v
        n_codes = 1 << p
        codes = np.arange(n_codes) if p <= 8 else np.unique(
            np.concatenate([[0, n_codes - 1], rng.integers(0, n_codes, 200)]))
        c0 = rng.uniform(-2, 2, R).astype(np.float32)
        b = rng.uniform(-2, 2, R).astype(np.float32)
        b[rng.random(R) < 0.3] = 0.0
        a = np.float32(rng.uniform(-2, 2))
        outs = []
        for code in codes:
            st, c = o.ref_kernel_apply(int(code), c0, a, b, lane=(w, p, v))
            assert st == 0
            outs.append(c)
        tag = f"ktl_{w}_{p}_{v}"
        fx[tag + "_codes"] = codes.astype(np.uint32)
        fx[tag + "_c0"], fx[tag + "_b"], fx[tag + "_a"] = c0, b, np.array([a], dtype=np.float32)
        fx[tag + "_out"] = np.stack(outs)
    for (w, p, v) in ((4, 8, 1), (2, 16, 1), (8, 8, 1)):
        R = w * p * v
        c0 = rng.uniform(-2, 2, R)
        b = rng.uniform(-2, 2, R) / 3.0  # full f64 mantissas
        a = rng.uniform(-2, 2) / 7.0
        codes = np.unique(np.concatenate([[0, (1 << p) - 1], rng.integers(0, 1 << p, 100)]))
        outs = []
        for code in codes:
            st, c = o.ref_kernel_apply_f64(int(code), c0, a, b, lane=(w, p, v))
            assert st == 0
            outs.append(c)
        tag = f"kt64_{w}_{p}_{v}"
        fx[tag + "_codes"] = codes.astype(np.uint32)
        fx[tag + "_c0"], fx[tag + "_b"], fx[tag + "_a"] = c0, b, np.array([a])
        fx[tag + "_out"] = np.stack(outs)
    mm_cases = [("f32", (4, 4, 4), 70, 150, 130), ("f32", (2, 16, 2), 40, 100, 200), ("f32", (1, 8, 1), 33, 70, 50),
                ("f64", (4, 8, 1), 64, 130, 100), ("f64", (8, 8, 1), 48, 96, 128), ("f64", (2, 4, 1), 30, 50, 41)]
    for t, (dt, lane, M, K, N) in enumerate(mm_cases):
        R = lane[0] * lane[1] * lane[2]
        ldb = (N + R - 1) // R * R
        A = o.gen_iid(M, K, seed=300 + t, mask_kind=1, p=0.7).astype(np.float64 if dt == "f64" else np.float32)
        B = o.gen_iid(K, N, seed=400 + t, mask_kind=2, p=0.6, block=max(1, lane[0] * lane[2]), ld=ldb)
        B = B.astype(np.float64 if dt == "f64" else np.float32)
        if dt == "f64":
            A = A / 3.0
            B = B / 7.0
        C = np.zeros((M, ldb), dtype=A.dtype)
        C[:, :N] = o.gen_iid(M, N, seed=500 + t).astype(A.dtype)
        C0 = C.copy()
        cnt = o.ref_multiply_lane(C, A, B, lane)
        tag = f"mml{t}"
        fx[tag + "_meta"] = np.array([1 if dt == "f64" else 0, *lane, M, K, N], dtype=np.int64)
        fx[tag + "_A"], fx[tag + "_B"], fx[tag + "_C0"], fx[tag + "_C"] = A, B, C0, C
        fx[tag + "_counters"] = np.array([cnt["kernel_invocations"], cnt["lane_fma_ops"], cnt["rows_skipped"],
                                          cnt["regions_skipped_by_zero_code"]], dtype=np.uint64)
    fx["mml_n"] = np.array([len(mm_cases)])

    # ---- MMMB bytes written by the reference writer
    path = os.path.join("/tmp", "golden_mmmb.bin")
    M4 = np.eye(4, dtype=np.float32) * np.float32(1.5)
    assert o.ref_lib().ref_write_matrix_f32(M4.ctypes.data, 4, 4, 4, path.encode()) == 0
    fx["mmmb_eye4"] = np.frombuffer(open(path, "rb").read(), dtype=np.uint8)

    np.savez_compressed(os.path.join(OUT, "reference_golden.npz"), **fx)
    print("wrote", os.path.join(OUT, "reference_golden.npz"), len(fx), "arrays")


if __name__ == "__main__":
    main()
