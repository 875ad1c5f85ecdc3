"""K2-TC time against the number of unit rounds (M rows, K = N = 4096): the intercept is the
kernel's fixed cost, the slope one round of units."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2402_14118_b200 as mmm  # noqa: E402
from paper_2402_14118_b200 import _native as N  # noqa: E402

zA, zB, bw = (float(sys.argv[1]), float(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else (0.6, 0.6, 8)
n = 4096
ctx = mmm.MmmContext(0)
ctx.set_algo(N.ALGO_TC)
b = torch.empty((n, n), dtype=torch.float32, device="cuda")
mmm.generate(b, seed=2, mask_kind=2, p=zB, block=bw, ctx=ctx)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for M in (768, 1536, 2304, 3072, 3840, 4096, 8192):
    a = torch.empty((M, n), dtype=torch.float32, device="cuda")
    c = torch.zeros((M, n), dtype=torch.float32, device="cuda")
    mmm.generate(a, seed=1, mask_kind=1, p=zA, ctx=ctx)
    ctx.preprocess(a, b)
    ts = []
    for it in range(5):
        e0.record()
        ctx.multiply(c, a, b, want_counters=False)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    units = (M + 255) // 256 * 22
    print(f"zA={zA} zB={zB} bw={bw} M={M}: units {units}  K2 {sorted(ts)[1]:.1f} us")
