"""Run one sweep cell through the TC path a few times (for ncu / timing)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2402_14118_b200 as mmm  # noqa: E402
from paper_2402_14118_b200 import _native as N  # noqa: E402

zA, zB, bw = (float(sys.argv[1]), float(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else (0.6, 0.6, 32)
algo = int(sys.argv[4]) if len(sys.argv) > 4 else N.ALGO_TC
n = 4096
ctx = mmm.MmmContext(0)
ctx.set_algo(algo)
a = torch.empty((n, n), dtype=torch.float32, device="cuda")
b = torch.empty((n, n), dtype=torch.float32, device="cuda")
c = torch.zeros((n, n), dtype=torch.float32, device="cuda")
mmm.generate(a, seed=1, mask_kind=1, p=zA, ctx=ctx)
mmm.generate(b, seed=2, mask_kind=2, p=zB, block=bw, ctx=ctx)
ctx.preprocess(a, b)
cnt = ctx.planned_counters()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for it in range(4):
    e0.record()
    ctx.multiply(c, a, b, want_counters=False)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"algo={algo} zA={zA} zB={zB} bw={bw}: {ms:.3f} ms  {2 * cnt.lane_fma_ops / ms / 1e9:.1f} TFLOP/s useful")
