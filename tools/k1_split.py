"""K1 on A only, B only and both for one 4096^2 sweep cell (for ncu launch lists)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2402_14118_b200 as mmm  # noqa: E402

n = 4096
ctx = mmm.MmmContext(0)
a = torch.empty((n, n), dtype=torch.float32, device="cuda")
b = torch.empty((n, n), dtype=torch.float32, device="cuda")
mmm.generate(a, seed=1, mask_kind=1, p=0.6, ctx=ctx)
mmm.generate(b, seed=2, mask_kind=2, p=0.6, block=8, ctx=ctx)
for it in range(3):
    ctx.preprocess(a, b)
    ctx.preprocess_a_only(a)
    ctx.preprocess_b_only(b)
torch.cuda.synchronize()
