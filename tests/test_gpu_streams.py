"""MmmStreams (independent multiplies on several contexts / CUDA streams) against the oracle.

Cells that overlap on the GPU (one cell's K1 chain beside another's K2: K2-TC leaves SMs free
and the K1 pass / pack CTAs take their tiles and items from atomic counters) must give the
results of the same cells run one after the other: AUTO within the north_star tolerance
 of the CPU oracle, and bit-identical to the single-context run (K2-TC's C update
has one writer per element); the exact path bit-identical to the oracle.
"""
import numpy as np
import pytest

from oracle import oracle as o  # noqa: F401

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2402_14118_b200 as mmm  # noqa: E402
from paper_2402_14118_b200 import _native as N  # noqa: E402

from test_gpu_parity import EXACT, bitexact, ctx, dev, gen_pair, run_gpu, run_oracle, within_tol  # noqa: E402,F401

CELLS = [(1024, 1024, 1024, 0.6, 0.6, 8), (512, 2048, 768, 0.9, 0.95, 32), (1024, 1024, 1024, 0.95, 0.8, 16),
         (300, 1000, 520, 0.7, 0.9, 8), (1024, 1024, 1024, 0.8, 0.9, 32), (2048, 512, 1024, 0.6, 0.95, 16)]


@pytest.mark.parametrize("nl,algo", [(2, N.ALGO_AUTO), (3, N.ALGO_AUTO), (2, EXACT)])
def test_streams_match_serial_and_oracle(ctx, nl, algo):
    pool = mmm.MmmStreams(nl, 0)
    for cx in pool.contexts:
        cx.set_algo(algo)
    ops, outs = [], []
    for i, (M, K, N_, zA, zB, bw) in enumerate(CELLS):
        A, B = gen_pair(100 + i, M, K, N_, zA, zB, bw)
        a = dev(A)[:, :K] if K != A.shape[1] else dev(A)
        b = dev(B)[:, :N_] if N_ != B.shape[1] else dev(B)
        cfull = torch.zeros((M, B.shape[1]), dtype=torch.float32, device="cuda")
        ops.append((A, B, a, b))
        outs.append((cfull, cfull[:, :N_] if N_ != B.shape[1] else cfull))
    for rep in range(3):  # repeated rounds: plans, scratch halves and counters are reused per stream
        for cfull, _ in outs:
            cfull.zero_()
        pool.run([(c, a, b) for (_, _, a, b), (_, c) in zip(ops, outs)])
        torch.cuda.synchronize()
    for (A, B, a, b), (cfull, c) in zip(ops, outs):
        C = cfull.cpu().numpy()
        Cr, _ = run_oracle(A, B)
        if algo == EXACT:
            assert bitexact(C, Cr)
        else:
            ok, worst = within_tol(C, Cr, A, B)
            assert ok, worst
            Cs, _ = run_gpu(ctx, A, B, algo=algo, N_=c.shape[1])
            assert bitexact(C, Cs), "streams differ from the single-context run"
    ctx.set_algo(N.ALGO_AUTO)
    pool.close()
