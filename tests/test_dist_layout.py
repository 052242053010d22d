"""Host-side logic of the multi-GPU path (no GPU): the block-cyclic layout of
include/randutv.h (C ABI queries vs the Python helpers vs brute force), and a
world_size-2 gloo run of the shard / gather plumbing the bench uses."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1703_00998_b200 import dist as D


def brute_owner_cols(n, b, P):
    owner = {}
    for c in range(n):
        owner.setdefault((c // b) % P, []).append(c)
    return owner


@pytest.mark.parametrize("n,b,P", [(1, 1, 1), (10, 3, 2), (500, 50, 3), (10000, 256, 8), (8000, 256, 8),
                                   (97, 13, 5), (30, 64, 4)])
def test_layout_matches_brute_force(n, b, P):
    owner = brute_owner_cols(n, b, P)
    tot = 0
    for r in range(P):
        cols = D.global_cols(n, b, r, P)
        assert list(cols) == owner.get(r, [])
        assert D.local_cols(n, b, r, P) == len(cols)
        for lc, gc in enumerate(cols):
            assert D._lib().randutv_dist_global_col(lc, b, r, P) == gc
        tot += len(cols)
    assert tot == n


def test_layout_rejects_bad_arguments():
    L = D._lib()
    assert L.randutv_dist_local_cols(10, 0, 0, 1) == -1
    assert L.randutv_dist_local_cols(10, 2, 3, 3) == -1
    assert L.randutv_dist_global_col(-1, 2, 0, 1) == -1


def test_shard_assemble_roundtrip_cpu():
    rng = np.random.default_rng(0)
    A = torch.from_numpy(rng.standard_normal((37, 101)))
    for P in (1, 2, 3, 7):
        shards = [D.shard(A, 8, r, P) for r in range(P)]
        assert all(S.stride(0) == 1 for S in shards if S.shape[1] > 1)
        np.testing.assert_array_equal(D.assemble(shards, 101, 8).numpy(), A.numpy())


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n, m, b = 53, 11, 4
        A = torch.arange(m * n, dtype=torch.float64).reshape(m, n)  # same on every rank
        S = D.shard(A, b, rank, world)
        # gather shard widths, pad, all_gather, reassemble on every rank
        w = torch.tensor([S.shape[1]])
        ws = [torch.zeros_like(w) for _ in range(world)]
        dist.all_gather(ws, w)
        wmax = int(max(x.item() for x in ws))
        pad = torch.zeros(m, wmax, dtype=torch.float64)
        pad[:, : S.shape[1]] = S
        pads = [torch.zeros_like(pad) for _ in range(world)]
        dist.all_gather(pads, pad)
        shards = [pads[r][:, : int(ws[r].item())] for r in range(world)]
        full = D.assemble([s.t().contiguous().t() for s in shards], n, b)
        ok = bool(torch.equal(full, A)) and sum(int(x.item()) for x in ws) == n
        # the max-over-ranks timing reduction bench.py uses
        t = torch.tensor([float(rank + 1)])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ok = ok and t.item() == float(world)
        out[rank] = 1 if ok else 0
    finally:
        dist.destroy_process_group()


def test_gloo_world2_shard_gather():
    world = 2
    port = 29500 + (os.getpid() % 1000)
    res = torch.zeros(world, dtype=torch.int32).share_memory_()
    mp.spawn(_worker, args=(world, port, res), nprocs=world, join=True)
    assert res.tolist() == [1] * world
