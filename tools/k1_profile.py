"""Run K1 (preprocess) on one 4096^3 sweep cell a few times, AUTO plan (for ncu / timing)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2402_14118_b200 as mmm  # noqa: E402

zA, zB, bw = (float(sys.argv[1]), float(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else (0.6, 0.6, 8)
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 4
n = 4096
ctx = mmm.MmmContext(0)
a = torch.empty((n, n), dtype=torch.float32, device="cuda")
b = torch.empty((n, n), dtype=torch.float32, device="cuda")
mmm.generate(a, seed=1, mask_kind=1, p=zA, ctx=ctx)
mmm.generate(b, seed=2, mask_kind=2, p=zB, block=bw, ctx=ctx)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for it in range(reps):
    flush.zero_()
    e0.record()
    ctx.preprocess(a, b)
    e1.record()
    torch.cuda.synchronize()
    print(f"K1 zA={zA} zB={zB} bw={bw}: {e0.elapsed_time(e1) * 1e3:.1f} us")
