import sys, numpy as np, torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import paper_2402_14118_b200 as mmm
from paper_2402_14118_b200 import _native as N
from oracle import oracle as o
import test_gpu_parity as T
A, B = T.gen_pair(2, 4096, 4096, 4096, 0.6, 0.6, 8)
bits_ref = o.a_bitmap(A, K=4096)
codes_ref = o.pattern_codes(B).astype(np.uint8)
a, b = T.dev(A), T.dev(B)
nbad = 0
for it in range(30):
    ctx = mmm.MmmContext(0)
    ctx.preprocess(a, b)
    bits = ctx.export_a_bitmap(4096, 4096)
    codes = ctx.export_b_codes(4096, B.shape[1])
    okb = np.array_equal(bits, bits_ref); okc = np.array_equal(codes, codes_ref)
    if not (okb and okc):
        nbad += 1
        rows = np.unique(np.argwhere(bits != bits_ref)[:, 0]).tolist()
        print(it, "bits", okb, "codes", okc, rows[:10], flush=True)
    del ctx
print("bad runs", nbad)
