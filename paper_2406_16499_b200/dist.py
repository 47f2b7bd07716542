"""Multi-GPU plumbing for the batched path.

Only the batched workload partitions: problems are independent, so rank r
owns a contiguous slice of the global batch and solves it with no data-path
collective.  The only cross-rank traffic is bookkeeping (max-over-ranks
timing) and an optional final gather of the results to rank 0 -- one
collective over NCCL (NVLink/NVSwitch) on GPUs, gloo in the CPU tests.
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    start: int   # first global problem index owned by this rank
    count: int   # problems owned by this rank
    seed: int    # generator seed of this rank's slice


def shard_plan(total: int, world: int, rank: int, base_seed: int = 1000) -> Shard:
    """Contiguous near-equal split of `total` problems over `world` ranks."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    q, r = divmod(total, world)
    count = q + (1 if rank < r else 0)
    start = rank * q + min(rank, r)
    return Shard(rank, world, start, count, base_seed + start)


def weak_plan(per_rank: int, world: int, rank: int, base_seed: int = 1000) -> Shard:
    """Weak scaling: every rank owns `per_rank` problems of a world*per_rank batch."""
    return Shard(rank, world, rank * per_rank, per_rank, base_seed + rank * per_rank)


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (device time) over all ranks; identity without a group."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_rows_to_rank0(t, counts):
    """Concatenate every rank's (count_r, ...) tensor on rank 0 in rank order
    (the final result gather).  Returns the full tensor on rank 0, None elsewhere."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return t
    world = dist.get_world_size()
    width = max(counts)
    pad = torch.zeros((width,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
    pad[: t.shape[0]] = t
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad)
    if dist.get_rank() != 0:
        return None
    return torch.cat([b[:c] for b, c in zip(bufs, counts)], dim=0)
