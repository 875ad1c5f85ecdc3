"""Quick TC-path correctness probe: K2-TC vs the CPU oracle (tolerance 1e-5 * Σ|a||b|)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2402_14118_b200 as mmm  # noqa: E402
from paper_2402_14118_b200 import _native as N  # noqa: E402
from oracle import oracle as o  # noqa: E402


def case(ctx, M, K, Nn, zA, zB, bw, seed=1):
    ld = mmm.round_up(K, 64)
    A = o.gen_iid(M, K, mmm.matrix_seed(seed, "A"), mask_kind=1, p=zA, ld=ld)
    ldb = mmm.round_up(Nn, 64)
    B = o.gen_iid(K, Nn, mmm.matrix_seed(seed, "B"), mask_kind=2, p=zB, block=bw, ld=ldb)
    a = torch.from_numpy(A).cuda()[:, :K]
    b = torch.from_numpy(B).cuda()[:, :Nn]
    c = torch.zeros((M, ldb), dtype=torch.float32, device="cuda")
    ctx.set_algo(N.ALGO_TC)
    ctx.preprocess(a, b)
    torch.cuda.synchronize()
    t0 = time.time()
    mmm.multiply_mmm(ctx, c[:, :Nn], a, b)
    torch.cuda.synchronize()
    dt = time.time() - t0
    Cg = c.cpu().numpy()
    Cr = np.zeros_like(Cg)
    o.multiply_mmm(Cr, np.ascontiguousarray(A[:, :K]), B)
    bad, worst = o.check_tolerance(Cg, Cr, np.ascontiguousarray(A[:, :K]), B, tol=1e-5)
    print(f"M={M} K={K} N={Nn} zA={zA} zB={zB} bw={bw}: bad={bad} worst={worst:.3e} "
          f"maxabs={np.abs(Cg - Cr).max():.3e} t={dt * 1e3:.2f} ms", flush=True)
    return bad == 0


if __name__ == "__main__":
    ctx = mmm.MmmContext(0)
    ok = True
    for args in [(128, 32, 256, 0.0, 0.0, 16), (128, 64, 256, 0.5, 0.5, 16), (256, 256, 512, 0.8, 0.8, 16),
                 (1024, 1024, 1024, 0.8, 0.8, 16), (100, 77, 130, 0.6, 0.6, 8), (4096, 4096, 4096, 0.8, 0.8, 16),
                 (4096, 4096, 4096, 0.6, 0.6, 32)]:
        ok &= case(ctx, *args)
    print("ALL OK" if ok else "FAIL")
