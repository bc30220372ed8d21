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


def _slice_flops(fix, size, F):
    """Algorithmic FLOPs of the frames with these fixations: oracle plans (the checker) fed to
    the product's accounting (costs.batch_flops), as bench.py does with device plans."""
    from oracle import fovea_oracle as fo
    from paper_2012_08655_b200 import costs

    cap = (size[0] // F + 2) * (size[1] // F + 2)
    lengths = np.ones((len(fix), cap), np.int32)
    meta = np.zeros((len(fix), 8), np.int32)
    for i, (x, y) in enumerate(fix):
        pl = fo.np_plan(size, fo.OracleParams(fragment_size=F, fixation=(float(x), float(y))))
        gh, gw = pl["length"].shape
        lengths[i, :gw * gh] = pl["length"].reshape(-1)
        meta[i, :4] = (pl["shift"][0], pl["shift"][1], gw, gh)
    return costs.batch_flops(size, F, 3, lengths, meta) if len(fix) else 0.0


def _cost_worker(rank, world, port, n_frames, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # the strong-scaling split of bench.py: one fixed batch, rank r owns shard_range(n, r, g)
        rng = np.random.default_rng(1)
        fix = np.stack([rng.integers(0, 256, n_frames), rng.integers(0, 256, n_frames)], axis=1)
        a, b = fk.shard_range(n_frames, rank, world)
        mine = torch.tensor([_slice_flops(fix[a:b], (256, 256), 32), float(b - a)], dtype=torch.float64)
        dist.all_reduce(mine)                      # test-only: the data path has no collective
        if rank == 0:
            q.put(dict(sum=float(mine[0]), frames=int(mine[1]),
                       whole=_slice_flops(fix, (256, 256), 32)))
    finally:
        dist.destroy_process_group()


def test_two_ranks_account_for_the_whole_batch_work():
    """Each rank plans and costs ITS slice of one fixed batch (BASELINE config 4's fixations);
    the per-rank algorithmic FLOPs add up to the whole batch's exactly: frames are independent,
    and a rank's roofline numerator is its slice's."""
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    n = 37
    mp.spawn(_cost_worker, args=(2, _free_port(), n, q), nprocs=2, join=True)
    got = q.get()
    assert got["frames"] == n
    assert got["sum"] == got["whole"] > 0


def test_bench_fixation_track_stays_inside_the_frame():
    import bench

    fix = bench.moving_fixations(256)
    assert fix.shape == (256, 2) and fix.dtype == np.float64
    assert fix[:, 0].min() >= 0 and fix[:, 0].max() < 1920
    assert fix[:, 1].min() >= 0 and fix[:, 1].max() < 1080
    assert tuple(fix[0]) == (1728.0, 540.0)
