"""Scenario sharding across ranks (one process per GPU) and the timing
reduction bench.py uses.  The path has no data exchange: each rank solves
its own contiguous shard; only the step time is reduced (max over ranks)."""

from __future__ import annotations


def shard_range(rank, world, per_rank, total):
    """[start, stop) of rank's shard: weak scaling, per_rank scenarios each,
    wrapping around a table of `total` scenarios."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    start = (rank * per_rank) % total
    return start, start + per_rank


def max_over_ranks(value, dist=None, device=None):
    """Max of a scalar over all ranks (the contract's multi-GPU timing rule)."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_results(arrays, dist=None, device=None):
    """Concatenate per-rank result arrays on every rank (all_gather; optional,
    outside any timed region)."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return arrays
    import torch
    out = []
    for a in arrays:
        t = torch.as_tensor(a, device=device)
        parts = [torch.empty_like(t) for _ in range(dist.get_world_size())]
        dist.all_gather(parts, t)
        out.append(torch.cat(parts).cpu().numpy())
    return out
