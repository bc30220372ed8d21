"""world_size-2 gloo checks of the multi-GPU host logic: frames shard
contiguously with no data-path collective; the bench takes the max time over ranks and
sums the per-rank frame counts."""

import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2012_08655_b200 as fk


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n_frames, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        a, b = fk.shard_range(n_frames, rank, world)
        # every rank derives the same synthetic batch from the seed and owns frames [a, b)
        fix = np.random.default_rng(0).uniform(0, 256, (n_frames, 2))
        owned = torch.zeros(n_frames, dtype=torch.int64)
        owned[a:b] = 1
        checksum = torch.tensor([float(fix[a:b].sum())], dtype=torch.float64)
        elapsed = torch.tensor([1.0 + rank], dtype=torch.float64)    # rank 1 is "slower"
        dist.all_reduce(owned)                                       # test-only bookkeeping
        dist.all_reduce(checksum)
        dist.all_reduce(elapsed, op=dist.ReduceOp.MAX)
        count = torch.tensor([b - a], dtype=torch.int64)
        dist.all_reduce(count)
        if rank == 0:
            q.put(dict(owned=owned.tolist(), checksum=float(checksum), elapsed=float(elapsed),
                       count=int(count), total=float(fix.sum())))
    finally:
        dist.destroy_process_group()


def test_two_ranks_partition_the_batch_exactly_once():
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    n = 257
    mp.spawn(_worker, args=(2, _free_port(), n, q), nprocs=2, join=True)
    got = q.get()
    assert got["owned"] == [1] * n             # every frame owned by exactly one rank
    assert got["count"] == n
    assert abs(got["checksum"] - got["total"]) < 1e-6
    assert got["elapsed"] == 2.0               # max over ranks, as bench.py reports


def test_bench_fixation_track_stays_inside_the_frame():
    import bench

    fix = bench.moving_fixations(256)
    assert fix.shape == (256, 2) and fix.dtype == np.float64
    assert fix[:, 0].min() >= 0 and fix[:, 0].max() < 1920
    assert fix[:, 1].min() >= 0 and fix[:, 1].max() < 1080
    assert tuple(fix[0]) == (1728.0, 540.0)
