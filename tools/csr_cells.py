"""K2 time of AUTO vs forced K2-CSR / K2-TC / K2-SIMT on sweep cells and configs[3] (cost-model calibration)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2402_14118_b200 as mmm  # noqa: E402
from paper_2402_14118_b200 import _native as N  # noqa: E402

T95 = 1.6448536269514722
cells = [(4096, 4096, 4096, 0.6, 0.6, 8), (4096, 4096, 4096, 0.95, 0.6, 8), (4096, 4096, 4096, 0.95, 0.95, 8),
         (4096, 4096, 4096, 0.9, 0.9, 16), (4096, 4096, 4096, 0.95, 0.95, 32), (4096, 4096, 4096, 0.8, 0.9, 32),
         ("cfg4",)]
ctx = mmm.MmmContext(0)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
names = {N.ALGO_AUTO: "auto", N.ALGO_CSR: "csr", N.ALGO_TC: "tc", N.ALGO_SIMT_BCAST: "simt"}
for cell in cells:
    if cell[0] == "cfg4":
        M, K, Nn = 64, 12288, 49152
        a = torch.empty((M, K), dtype=torch.float32, device="cuda")
        b = torch.empty((K, Nn), dtype=torch.float32, device="cuda")
        mmm.generate(a, seed=1, value_kind=2, thresh=T95, ctx=ctx)
        mmm.generate(b, seed=2, value_kind=1, sigma=0.02, mask_kind=2, p=0.85, block=16, ctx=ctx)
        label = "cfg4"
    else:
        M, K, Nn, zA, zB, bw = cell
        a = torch.empty((M, K), dtype=torch.float32, device="cuda")
        b = torch.empty((K, Nn), dtype=torch.float32, device="cuda")
        mmm.generate(a, seed=1, mask_kind=1, p=zA, ctx=ctx)
        mmm.generate(b, seed=2, mask_kind=2, p=zB, block=bw, ctx=ctx)
        label = f"zA={zA} zB={zB} bw={bw}"
    c = torch.zeros((M, Nn), dtype=torch.float32, device="cuda")
    out = []
    for algo in (N.ALGO_AUTO, N.ALGO_CSR, N.ALGO_TC, N.ALGO_SIMT_BCAST):
        ctx.set_algo(algo)
        ts, t1 = [], []
        for it in range(4):
            e0.record()
            ctx.preprocess(a, b)
            e1.record()
            torch.cuda.synchronize()
            t1.append(e0.elapsed_time(e1) * 1e3)
            e0.record()
            ctx.multiply(c, a, b, want_counters=False)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        extra = f"[{names.get(ctx.last_algo(), ctx.last_algo())}]" if algo == N.ALGO_AUTO else ""
        out.append(f"{names[algo]}{extra} K1 {sorted(t1)[1]:.0f} K2 {sorted(ts)[1]:.0f}")
    print(label, " | ".join(out), flush=True)
    del a, b, c
    torch.cuda.empty_cache()
