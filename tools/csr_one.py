"""One forced K2-CSR multiply on configs[3] (for ncu)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2402_14118_b200 as mmm  # noqa: E402
from paper_2402_14118_b200 import _native as N  # noqa: E402

M, K, Nn = 64, 12288, 49152
ctx = mmm.MmmContext(0)
a = torch.empty((M, K), dtype=torch.float32, device="cuda")
b = torch.empty((K, Nn), dtype=torch.float32, device="cuda")
mmm.generate(a, seed=1, value_kind=2, thresh=1.6448536269514722, ctx=ctx)
mmm.generate(b, seed=2, value_kind=1, sigma=0.02, mask_kind=2, p=0.85, block=16, ctx=ctx)
c = torch.zeros((M, Nn), dtype=torch.float32, device="cuda")
ctx.set_algo(N.ALGO_CSR)
ctx.preprocess(a, b)
for _ in range(2):
    ctx.multiply(c, a, b, want_counters=False)
torch.cuda.synchronize()
print("ok")
