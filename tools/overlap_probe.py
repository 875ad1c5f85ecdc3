"""Sweep step on 1 context / stream vs cells dealt round-robin to S contexts on S streams
(the K1 chain of one cell fills the tail round and the single-CTA phases of another's K2)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2402_14118_b200 as mmm

dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
wl = sys.argv[1] if len(sys.argv) > 1 else "sweep"
cells = bench.workload_cells(wl)
ctx0 = mmm.MmmContext(0)
As, Bs, _ = bench.make_inputs(cells, ctx0, 0, 1, torch, None, dev)
for S in (1, 2, 3, 4, 1, 2):
    ctxs = [mmm.MmmContext(0) for _ in range(S)]
    streams = [torch.cuda.Stream(dev) for _ in range(S)]
    Cs = [{} for _ in range(S)]
    for s in range(S):
        for (_, M, K, N, sa, sb) in cells:
            if (M, N) not in Cs[s]:
                Cs[s][(M, N)] = torch.zeros((M, mmm.round_up(N, 64)), dtype=torch.float32, device=dev)[:, :N]

    def step():
        for t, (label, M, K, N, sa, sb) in enumerate(cells):
            s = t % S
            with torch.cuda.stream(streams[s]):
                a, b = As[sa["key"]], Bs[sb["key"]]
                ctxs[s].preprocess(a, b)
                ctxs[s].multiply(Cs[s][(M, N)], a, b, want_counters=False)

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    main = torch.cuda.current_stream(dev)
    e0.record(main)
    for st in streams:
        st.wait_event(e0)
    n = 5
    for _ in range(n):
        step()
    for st in streams:
        main.wait_stream(st)
    e1.record(main)
    torch.cuda.synchronize()
    print(f"{wl}: {S} stream(s): {e0.elapsed_time(e1) / n:.3f} ms/step", flush=True)
    del ctxs, Cs
    torch.cuda.empty_cache()
