"""Multi-process (world_size 2, gloo, CPU) coverage of the batched path's
sharding, max-over-ranks timing and final result gather."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2406_16499_b200.dist import gather_rows_to_rank0, max_over_ranks, shard_plan, weak_plan


def test_shard_plan_covers_batch_exactly():
    for total in (1, 7, 65536, 65537):
        for world in (1, 2, 4, 8):
            shards = [shard_plan(total, world, r) for r in range(world)]
            assert sum(s.count for s in shards) == total
            assert [s.start for s in shards] == [sum(x.count for x in shards[:r]) for r in range(world)]
            assert max(s.count for s in shards) - min(s.count for s in shards) <= 1


def test_weak_plan():
    s = weak_plan(65536, 8, 3)
    assert (s.start, s.count, s.seed) == (3 * 65536, 65536, 1000 + 3 * 65536)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, total, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.oracle import Oracle
        from paper_2406_16499_b200 import generate as G

        sh = shard_plan(total, world, rank)
        # every rank solves its own slice (the CPU oracle stands in for the device here)
        A, B, b, d, _ = G.lse_batch_numpy(sh.count, 12, 6, 2, seed=1000 + sh.start)
        x, *_ = Oracle("port").mplse_batch(A, B, b, d)
        tmax = max_over_ranks(float(rank + 1))
        counts = [shard_plan(total, world, r).count for r in range(world)]
        full = gather_rows_to_rank0(torch.from_numpy(x), counts)
        if rank == 0:
            np.save(os.path.join(out_dir, "x.npy"), full.numpy())
            np.save(os.path.join(out_dir, "tmax.npy"), np.array([tmax]))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_shard_solve_gather(tmp_path, port):
    total = 7
    mp.spawn(_worker, args=(2, _free_port(), total, str(tmp_path)), nprocs=2, join=True)
    x = np.load(tmp_path / "x.npy")
    assert np.load(tmp_path / "tmax.npy")[0] == 2.0
    # identical to a single-process solve of the whole batch (per-problem seeds)
    from paper_2406_16499_b200 import generate as G

    xs = []
    for r in range(2):
        sh = shard_plan(total, 2, r)
        A, B, b, d, _ = G.lse_batch_numpy(sh.count, 12, 6, 2, seed=1000 + sh.start)
        xs.append(port.mplse_batch(A, B, b, d)[0])
    assert np.array_equal(x, np.concatenate(xs))
    A, B, b, d, _ = G.lse_batch_numpy(total, 12, 6, 2, seed=1000)
    assert np.array_equal(x, port.mplse_batch(A, B, b, d)[0])


def _gpu_worker(rank, world, port, total, out_dir):
    """One rank of the sharded batch on the GPU: generate only the shard (per-block
    seeds), solve it through mplse_batched, gather to rank 0 (gloo over host
    copies: both ranks share the one GPU of the test box, and neither waits on
    the other's kernels)."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2406_16499_b200 as P
        from paper_2406_16499_b200 import generate as G

        torch.cuda.set_device(0)
        sh = shard_plan(total, world, rank)
        A, B, b, d, _ = G.lse_batch_torch(sh.count, 256, 128, 32, seed=1000, device="cuda", start=sh.start)
        out = P.mplse_batched(A, B, b, d)
        torch.cuda.synchronize()
        counts = [shard_plan(total, world, r).count for r in range(world)]
        full = gather_rows_to_rank0(out.x.cpu(), counts)
        its = gather_rows_to_rank0(out.iterations.cpu(), counts)
        if rank == 0:
            np.save(os.path.join(out_dir, "x.npy"), full.numpy())
            np.save(os.path.join(out_dir, "it.npy"), its.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_two_rank_gpu_shards_match_single_gpu(tmp_path, gpu):
    """the sharded batch, gathered, is bitwise the single-GPU solve."""
    total = 3000  # shards straddle a generator block boundary (1024)
    mp.spawn(_gpu_worker, args=(2, _free_port(), total, str(tmp_path)), nprocs=2, join=True)
    from paper_2406_16499_b200 import generate as G

    A, B, b, d, _ = G.lse_batch_torch(total, 256, 128, 32, seed=1000, device="cuda")
    out = gpu.mplse_batched(A, B, b, d)
    assert np.array_equal(np.load(tmp_path / "x.npy"), out.x.cpu().numpy())
    assert np.array_equal(np.load(tmp_path / "it.npy"), out.iterations.cpu().numpy())
