"""K1 timing (and the path AUTO picks) on a cfg4-shaped B (12288 x 49152, 16-wide blocks
kept 0.15) and a sweep cell."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2402_14118_b200 as mmm
ctx = mmm.MmmContext(0)
for (M, K, N, zA, zB, bw) in [(64, 12288, 49152, 0.95, 0.85, 16), (4096, 4096, 4096, 0.6, 0.6, 8)]:
    a = torch.empty((M, K), dtype=torch.float32, device="cuda")
    b = torch.empty((K, N), dtype=torch.float32, device="cuda")
    c = torch.zeros((M, N), dtype=torch.float32, device="cuda")
    mmm.generate(a, seed=1, mask_kind=1, p=zA, ctx=ctx)
    mmm.generate(b, seed=2, mask_kind=2, p=zB, block=bw, ctx=ctx)
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    for it in range(4):
        e0.record(); ctx.preprocess(a, b); e1.record(); ctx.multiply(c, a, b, want_counters=False); e2.record()
        torch.cuda.synchronize()
    print(f"{M}x{K}x{N}: K1 {e0.elapsed_time(e1) * 1e3:.0f} us  K2 {e1.elapsed_time(e2) * 1e3:.0f} us  path {ctx.last_algo()}",
          flush=True)
    del a, b, c
