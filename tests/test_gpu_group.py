"""Multi-GPU entry points (mmmcu_group_*, csrc/mmmcu_group.cu).

gpurun offers one B200, so the multi-rank logic is exercised two ways: a 1-GPU group runs the
real NCCL path (ncclCommInitAll + ncclBroadcast), and groups that repeat device 0 run the
same partition / replica / per-rank plan logic with device-copy replicas.  Every shard is
compared with the CPU oracle: bit-exact under EXACT, tolerance under AUTO.
"""
import numpy as np
import pytest

from oracle import oracle as o

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2402_14118_b200 as mmm  # noqa: E402
from paper_2402_14118_b200 import _native as N  # noqa: E402

from test_gpu_parity import TOL, EXACT, bitexact, dev, gen_pair, within_tol  # noqa: E402


@pytest.fixture(scope="module")
def cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def row_shards(A, g, K):
    M = A.shape[0]
    out = []
    for r in range(g):
        r0, r1 = mmm.shard_rows(M, g, r)
        out.append(dev(A[r0:r1])[:, :K])
    return out


@pytest.mark.parametrize("g", [1, 3, 8])
@pytest.mark.parametrize("algo", [EXACT, N.ALGO_AUTO])
def test_row_sharded_matches_oracle(cuda, g, algo):
    M, K, N_ = 1000, 768, 640
    A, B = gen_pair(51, M, K, N_, 0.8, 0.8, 16)
    grp = mmm.MmmGroup([0] * g)
    assert grp.size == g
    assert grp.uses_nccl == (g == 1)  # a repeated device replicates with device copies
    grp.set_algo(algo)
    a_sh = row_shards(A, g, K)
    c_sh = [torch.zeros((a.shape[0], N_), dtype=torch.float32, device="cuda") for a in a_sh]
    cnt = grp.multiply_sharded(c_sh, a_sh, dev(B), version_a=1, version_b=1)
    Cr = np.zeros((M, N_), np.float32)
    ocnt = o.multiply_mmm(Cr, np.ascontiguousarray(A[:, :K]), B)
    C = np.concatenate([c.cpu().numpy() for c in c_sh])
    if algo == EXACT:
        assert bitexact(C, Cr)
    else:
        ok, worst = within_tol(C, Cr, A, B)
        assert ok and worst < 0.5 * TOL, worst
    assert cnt.lane_fma_ops == ocnt["lane_fma_ops"]
    assert cnt.kernel_invocations == ocnt["kernel_invocations"]
    assert cnt.rows_skipped == ocnt["rows_skipped"]
    grp.close()


def test_row_sharded_plan_reuse_and_accumulate(cuda):
    # a second call with the same operands and versions skips the broadcast and the K1 pass
    # and accumulates again (c += a*b): the oracle chain continued from the first result
    M, K, N_ = 512, 512, 512
    A, B = gen_pair(52, M, K, N_, 0.7, 0.8, 8)
    grp = mmm.MmmGroup([0, 0])
    grp.set_algo(EXACT)
    a_sh = row_shards(A, 2, K)
    b = dev(B)
    c_sh = [torch.zeros((a.shape[0], N_), dtype=torch.float32, device="cuda") for a in a_sh]
    grp.multiply_sharded(c_sh, a_sh, b, 7, 9)
    grp.multiply_sharded(c_sh, a_sh, b, 7, 9)
    assert grp.broadcast_ms == 0.0
    Cr = np.zeros((M, N_), np.float32)
    o.multiply_mmm(Cr, np.ascontiguousarray(A[:, :K]), B)
    o.multiply_mmm(Cr, np.ascontiguousarray(A[:, :K]), B)
    assert bitexact(np.concatenate([c.cpu().numpy() for c in c_sh]), Cr)
    grp.close()


@pytest.mark.parametrize("g", [1, 3])
def test_col_sharded_skinny(cuda, g):
    # configs[3]-shaped (skinny M): B / C split by 64-column slabs, A broadcast
    M, K, N_ = 64, 1536, 1000
    A, B = gen_pair(53, M, K, N_, 0.95, 0.85, 16)
    grp = mmm.MmmGroup([0] * g)
    grp.set_algo(EXACT)
    slabs = []
    ld = mmm.round_up(mmm.shard_cols(N_, g, 0)[1], 64)  # one leading dimension for every slab
    for r in range(g):
        c0, c1 = mmm.shard_cols(N_, g, r)
        slabs.append(torch.zeros((M, ld), dtype=torch.float32, device="cuda")[:, : c1 - c0])
    cnt = grp.multiply_sharded_cols(slabs, dev(A)[:, :K], dev(B)[:, :N_], 3, 4)
    Cr = np.zeros((M, B.shape[1]), np.float32)
    ocnt = o.multiply_mmm(Cr, np.ascontiguousarray(A[:, :K]), B)
    C = np.concatenate([s.cpu().numpy() for s in slabs], axis=1)
    assert bitexact(C, Cr[:, :N_])
    assert cnt.lane_fma_ops == ocnt["lane_fma_ops"]
    grp.close()


def test_group_errors(cuda):
    with pytest.raises((mmm.MmmError, ValueError)):
        mmm.MmmGroup([0, 99])
    grp = mmm.MmmGroup([0])
    A, B = gen_pair(54, 64, 64, 64, 0.5, 0.5, 8)
    with pytest.raises(mmm.DimensionMismatchError):
        grp.multiply_sharded([torch.zeros((16, 64), device="cuda")], [dev(A)[:32]], dev(B))
    grp.close()
