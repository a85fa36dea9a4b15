"""Multi-GPU plumbing for the labeling path (one process per GPU, torch.distributed).

Batches shard by image: images are independent, so each rank
labels a contiguous block of the batch and no data-path collective is needed; only the
timing (max over ranks) and optional result checksums are reduced.
"""
from __future__ import annotations

import os
from dataclasses import dataclass


@dataclass(frozen=True)
class Rank:
    rank: int
    world: int
    local: int


def env_rank() -> Rank:
    return Rank(int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
                int(os.environ.get("LOCAL_RANK", "0")))


def shard_range(n_items: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous block [lo, hi) of n_items for `rank`; sizes differ by at most one."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(n_items, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def balanced_shards(costs: list[float], world: int) -> list[list[int]]:
    """Items -> ranks so that the ranks' summed costs are even (longest-processing-time
    greedy: items by decreasing cost, each to the currently lightest rank; ties go to the
    lower rank).  Deterministic, so every rank computes the same assignment without a
    collective.  Each rank's list is returned in ascending item order."""
    if world < 1:
        raise ValueError("bad world")
    load = [0.0] * world
    out: list[list[int]] = [[] for _ in range(world)]
    for i in sorted(range(len(costs)), key=lambda k: (-costs[k], k)):
        r = min(range(world), key=lambda q: (load[q], q))
        load[r] += costs[i]
        out[r].append(i)
    return [sorted(x) for x in out]


def image_cost(density: float, granularity: int) -> float:
    """Relative device cost of one generated image per pixel: a fixed part plus a part growing
    with the expected run density 2 d (1 - d) / g of the reference generator's g x g blocks
    (generator.hpp:46-83).  Fitted to the per-cell device times of the config-2 sweep on a
    B200 (tools/prof_driver.py --sweep: 13.1 + 116 (2d(1-d))^0.86 / g^1.6 us per 2048^2 image,
    within 23% on every cell)."""
    r = 2.0 * density * (1.0 - density)
    return 1.0 + 8.87 * r ** 0.86 / max(granularity, 1) ** 1.6


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (e.g. a CUDA-event time) over the process group."""
    import torch
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: int, device=None) -> int:
    import torch
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return int(value)
    t = torch.tensor([int(value)], dtype=torch.int64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return int(t.item())
