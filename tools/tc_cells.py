"""K2 time of a few sweep cells under AUTO (K1 excluded), for A/B timing of K2 variants."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2402_14118_b200 as mmm  # noqa: E402

cells = [(0.6, 0.6, 8), (0.6, 0.9, 16), (0.6, 0.95, 8), (0.6, 0.95, 32), (0.95, 0.95, 16)]
n = 4096
ctx = mmm.MmmContext(0)
a = torch.empty((n, n), dtype=torch.float32, device="cuda")
b = torch.empty((n, n), dtype=torch.float32, device="cuda")
c = torch.zeros((n, n), dtype=torch.float32, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for zA, zB, bw in cells:
    mmm.generate(a, seed=1, mask_kind=1, p=zA, ctx=ctx)
    mmm.generate(b, seed=2, mask_kind=2, p=zB, block=bw, ctx=ctx)
    ctx.preprocess(a, b)
    ts = []
    for it in range(5):
        e0.record()
        ctx.multiply(c, a, b, want_counters=False)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    print(f"zA={zA} zB={zB} bw={bw} path={ctx.last_algo()}: K2 {sorted(ts)[2]:.1f} us")
