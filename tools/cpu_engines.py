"""Time the two reference-kind CPU engines (oracle/_ref) on the same sweep-cell sample:
ref_multiply_parallel (row-wise, Fig. 4 A-skip) and ref_multiply_mmm (SPEC leaf-blocked,
ABlockIndex traversal)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as o  # noqa: E402

print(o.ref_so_path(), os.cpu_count())
for zA, zB, rows in ((0.6, 0.6, 256), (0.8, 0.8, 512), (0.95, 0.95, 2048)):
    A = o.gen_iid(rows, 4096, seed=1, mask_kind=1, p=zA)
    B = o.gen_iid(4096, 4096, seed=2, mask_kind=2, p=zB, block=16)
    for f in (o.ref_multiply_parallel, o.ref_multiply_mmm):
        C = np.zeros((rows, 4096), np.float32)
        t0 = time.perf_counter()
        c = f(C, A, B, workers=0)
        print(f"{f.__name__:24s} zA={zA} zB={zB} rows={rows}: {2 * c['lane_fma_ops'] / c['multiply_ns']:.2f} GFLOP/s "
              f"multiply {c['multiply_ns'] / 1e6:.1f} ms preprocess {c['preprocess_ns'] / 1e6:.1f} ms wall {time.perf_counter() - t0:.2f} s")
