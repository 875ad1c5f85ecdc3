"""K1 + K2 device times of one BASELINE config under each K2 algorithm (AUTO, SIMT, TC, CSR)."""
import sys
import time

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2402_14118_b200 as mmm  # noqa: E402
from paper_2402_14118_b200 import _native as N  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
cells = bench.workload_cells(name)
lab, M, K, Nn, sa, sb = cells[0]
dev = torch.device("cuda:0")
ctx = mmm.MmmContext(0)
ld = (Nn + 63) // 64 * 64
a = torch.empty((M, K), dtype=torch.float32, device=dev)
bfull = torch.zeros((K, ld), dtype=torch.float32, device=dev)
b = bfull[:, :Nn]
mmm.generate(a, seed=bench.seed_of(sa["key"]), value_kind=sa["value_kind"], sigma=sa["sigma"], thresh=sa["thresh"],
             mask_kind=sa["mask_kind"], p=sa["p"], block=sa["block"], ctx=ctx)
mmm.generate(b, seed=bench.seed_of(sb["key"]), value_kind=sb["value_kind"], sigma=sb["sigma"], thresh=sb["thresh"],
             mask_kind=sb["mask_kind"], p=sb["p"], block=sb["block"], ctx=ctx)
cfull = torch.zeros((M, ld), dtype=torch.float32, device=dev)
c = cfull[:, :Nn]
e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
for algo, nm in ((N.ALGO_AUTO, "auto"), (N.ALGO_SIMT_BCAST, "simt"), (N.ALGO_TC, "tc"), (N.ALGO_CSR, "csr")):
    ctx.set_algo(algo)
    for it in range(3):
        e[0].record()
        ctx.preprocess(a, b)
        e[1].record()
        ctx.multiply(c, a, b, want_counters=False)
        e[2].record()
        torch.cuda.synchronize()
    print(f"{name} {nm:5s}: K1 {e[0].elapsed_time(e[1]):.3f} ms  K2 {e[1].elapsed_time(e[2]):.3f} ms  (path {ctx.last_algo()})")
