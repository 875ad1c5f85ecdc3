"""Multi-rank plumbing of the sharded run on CPU with the gloo backend,
world_size 2: rank 0 generates B and broadcasts it once, each rank generates its own A/C row
shard (row-offset generator), computes its C rows (CPU oracle standing in for K1+K2, which
need a GPU), and rank 0 checks that the concatenated shards and the summed WorkCounters equal
the single-process result bit for bit."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, M, K, N, out_path):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle import oracle as o
    import paper_2402_14118_b200 as mmm

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    r0, r1 = mmm.shard_rows(M, world, rank)
    seedA, seedB = mmm.matrix_seed(5, "A"), mmm.matrix_seed(5, "B")
    A = o.gen_iid(r1 - r0, K, seedA, mask_kind=1, p=0.85, row0=r0)  # this rank's rows only
    B = torch.zeros((K, N), dtype=torch.float32)
    if rank == 0:
        B = torch.from_numpy(o.gen_iid(K, N, seedB, mask_kind=2, p=0.85, block=16))
    dist.broadcast(B, src=0)  # B is broadcast once
    Bn = B.numpy()
    C = np.zeros((r1 - r0, N), np.float32)
    cnt = o.multiply_mmm(C, A, Bn)
    counts = torch.tensor([cnt["kernel_invocations"], cnt["lane_fma_ops"], cnt["rows_skipped"],
                           cnt["regions_skipped_by_zero_code"]], dtype=torch.int64)
    dist.all_reduce(counts)  # job totals
    spans = [mmm.shard_rows(M, world, r) for r in range(world)]
    rows_max = max(b - a for a, b in spans)
    mine = torch.zeros((rows_max, N), dtype=torch.float32)  # gather needs equal shapes
    mine[: r1 - r0] = torch.from_numpy(C)
    parts = [torch.zeros((rows_max, N), dtype=torch.float32) for _ in range(world)] if rank == 0 else None
    dist.gather(mine, parts, dst=0)
    if rank == 0:
        np.save(out_path, np.concatenate([p.numpy()[: b - a] for p, (a, b) in zip(parts, spans)]))
        np.save(out_path + ".cnt.npy", counts.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_run_equals_single(tmp_path, world):
    from oracle import oracle as o
    import paper_2402_14118_b200 as mmm

    M, K, N = 257, 320, 192
    out = str(tmp_path / "c.npy")
    mp.start_processes(_worker, args=(world, _free_port(), M, K, N, out), nprocs=world, join=True,
                       start_method="spawn")
    A = o.gen_iid(M, K, mmm.matrix_seed(5, "A"), mask_kind=1, p=0.85)
    B = o.gen_iid(K, N, mmm.matrix_seed(5, "B"), mask_kind=2, p=0.85, block=16)
    C = np.zeros((M, N), np.float32)
    cnt = o.multiply_mmm(C, A, B)
    Cs = np.load(out)
    assert np.array_equal(Cs.view(np.uint32), C.view(np.uint32))
    assert np.load(out + ".cnt.npy").tolist() == [cnt["kernel_invocations"], cnt["lane_fma_ops"],
                                                   cnt["rows_skipped"], cnt["regions_skipped_by_zero_code"]]


def test_row_offset_generator_matches_full():
    # shard generation with row0 reproduces the rows of the full matrix (device generator
    # semantics: mmmcu_generate(row0) hashes global coordinates)
    from oracle import oracle as o

    full = o.gen_iid(100, 64, 9, mask_kind=1, p=0.5)
    part = o.gen_iid(37, 64, 9, mask_kind=1, p=0.5, row0=40)
    assert np.array_equal(full[40:77], part)
