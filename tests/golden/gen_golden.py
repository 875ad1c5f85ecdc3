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

    # ---- MMMB bytes written by the reference writer
    path = os.path.join("/tmp", "golden_mmmb.bin")
    M4 = np.eye(4, dtype=np.float32) * np.float32(1.5)
    assert o.ref_lib().ref_write_matrix_f32(M4.ctypes.data, 4, 4, 4, path.encode()) == 0
    fx["mmmb_eye4"] = np.frombuffer(open(path, "rb").read(), dtype=np.uint8)

    np.savez_compressed(os.path.join(OUT, "reference_golden.npz"), **fx)
    print("wrote", os.path.join(OUT, "reference_golden.npz"), len(fx), "arrays")


if __name__ == "__main__":
    main()
