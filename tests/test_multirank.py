"""World-size-2 checks of the multi-GPU plumbing on CPU (gloo): rank slices are
disjoint and cover the job, the max-over-ranks timing reduction, and the
cost-balanced device split."""
import os

import numpy as np
import pytest
import torch.multiprocessing as mp


def _worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2208_09985_b200 import shard
    first, count = shard.rank_range(rank, world, 100000)
    gathered = [None] * world
    dist.all_gather_object(gathered, (first, count))
    t = shard.max_over_ranks(1.5 + rank)
    dist.barrier()
    if rank == 0:
        out.put((gathered, t))
    dist.destroy_process_group()


def test_rank_slices_and_max_over_ranks_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 2000)
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    gathered, t = q.get(timeout=120)
    for p in ps:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert gathered == [(0, 100000), (100000, 100000)]
    assert t == 2.5


def test_cost_cuts_balance_and_cover():
    from paper_2208_09985_b200 import shard
    rng = np.random.default_rng(1)
    lens = rng.integers(100, 20000, size=5000)
    for parts in (1, 2, 4, 8):
        cuts = shard.cost_cuts(lens, parts)
        assert cuts[0] == 0 and cuts[-1] == len(lens)
        assert (np.diff(cuts) >= 0).all()
        costs = [lens[a:b].sum() for a, b in zip(cuts[:-1], cuts[1:])]
        assert max(costs) - min(costs) <= 2 * lens.max()
    with pytest.raises(ValueError):
        shard.rank_range(2, 2, 10)
