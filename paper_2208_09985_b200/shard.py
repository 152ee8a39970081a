"""Multi-GPU plumbing for the benchmark and batch drivers (K5).

Pairs are independent: no data-path collective. Under
torchrun a rank aligns its own contiguous slice of the generator (weak scaling);
in one process, sg_align_packed(devices=[...]) splits a batch with the C++ plan
that `plan` exposes (host.cu plan_shards). torch.distributed is used
only for the barrier and the max-over-ranks timing.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _ffi


def rank_range(rank: int, world: int, per_rank: int):
    """Weak scaling: rank r aligns pairs [r*per_rank, (r+1)*per_rank) of the generator."""
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world {world}")
    return rank * per_rank, per_rank


def plan(batch, n_devices: int):
    """The library's device split of a PackedBatch (sg_plan_shards): per pair its
    device slot and its position in that device's batch, and whether the shards
    are gathered (cost buckets + longest-first) or contiguous ranges."""
    from .aligner import _check
    n = batch.n
    shard = np.zeros(max(n, 1), np.int32)
    pos = np.zeros(max(n, 1), np.int64)
    gathered = C.c_int()
    _check(_ffi.load().sg_plan_shards(C.byref(batch.c), n_devices,
                                      shard.ctypes.data_as(C.c_void_p),
                                      pos.ctypes.data_as(C.c_void_p), C.byref(gathered)))
    return shard[:n], pos[:n], bool(gathered.value)


def members(shard, pos, d: int):
    """Input indices of device slot d's pairs, in that device's order."""
    idx = np.nonzero(shard == d)[0]
    return idx[np.argsort(pos[idx], kind="stable")]


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
