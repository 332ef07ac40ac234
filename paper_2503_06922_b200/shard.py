"""Scenario sharding across ranks (one process per GPU) and the timing
reduction bench.py uses.  The path has no data exchange: each rank solves
its own contiguous shard (or claims chunks from a dynamic queue); only the
step time is reduced (max over ranks) and the results gathered at the end
(SURVEY §8(e))."""

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


class ChunkQueue:
    """Dynamic cross-rank work queue: chunks of `chunk` scenarios of a `total`
    table claimed through an atomic counter in the process group's key-value
    store (one `add` per claim), so ranks that draw cheap scenarios take more
    chunks (frame counts vary 3-400 per scenario)."""

    def __init__(self, store, key, total, chunk):
        if chunk < 1:
            raise ValueError("chunk must be >= 1")
        self.store, self.key, self.total, self.chunk = store, key, int(total), int(chunk)

    def next(self):
        """[start, stop) of the next unclaimed chunk, or None when the table is exhausted."""
        i = int(self.store.add(self.key, 1)) - 1
        a = i * self.chunk
        if a >= self.total:
            return None
        return a, min(self.total, a + self.chunk)


def all_max(arrays, dist=None):
    """Element-wise max over ranks of int64 arrays (ranks fill the entries they
    solved and -1 elsewhere): the union of a dynamically chunked run."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return arrays
    import numpy as np
    import torch
    out = []
    for a in arrays:
        t = torch.tensor(np.asarray(a, dtype=np.int64))  # a copy: the reduction is in place
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        out.append(t.numpy())
    return out
