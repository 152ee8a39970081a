"""Multi-GPU plumbing for the benchmark and batch drivers (K5).

Pairs are independent: no data-path collective. A
rank aligns its own contiguous slice; torch.distributed is used only for the
barrier and the max-over-ranks timing.
"""
from __future__ import annotations

import numpy as np


def rank_range(rank: int, world: int, per_rank: int):
    """Weak scaling: rank r aligns pairs [r*per_rank, (r+1)*per_rank) of the generator."""
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world {world}")
    return rank * per_rank, per_rank


def cost_cuts(lengths, parts: int):
    """Contiguous shards of balanced cost (text+pattern length); mirrors the C ABI's
    device split (host.cu align_packed_impl). Returns parts+1 cut indices."""
    lengths = np.asarray(lengths, dtype=np.int64)
    n = len(lengths)
    cuts = np.zeros(parts + 1, dtype=np.int64)
    total = int(lengths.sum())
    acc = np.cumsum(lengths)
    d = 1
    for k in range(n):
        while d < parts and acc[k] * parts >= total * d:
            cuts[d] = k + 1
            d += 1
        if d >= parts:
            break
    while d < parts:
        cuts[d] = n
        d += 1
    cuts[parts] = n
    return cuts


def max_over_ranks(value: float, device=None) -> float:
    """Max of a float over the default process group (identity without one)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64,
                     device=device if device is not None else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
