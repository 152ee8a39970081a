"""Multi-GPU plumbing on CPU: the device split is the C++ plan behind
the C ABI (sg_plan_shards, host.cu plan_shards), exercised here without a GPU.

* world_size-2 gloo: each rank takes its shard of a cfg5 prefix from the ABI's plan,
  aligns it with the oracle (the CPU checker standing in for its GPU), and rank 0
  puts the results back in input order through the plan's permutation; the result
  must reproduce the reference's whole-config digest block (batch.cpp:28,45: outputs
  in input order). Also the rank slices and the max-over-ranks timing reduction.
* the plan itself: every pair in exactly one shard, positions a permutation, cfg5's
  mix bucketed and dealt longest-first, cfg3's uniform pairs contiguous, loads balanced.
"""
import os

import numpy as np
import pytest
import torch.multiprocessing as mp

N_CFG5 = 1000  # digest block 0 of tests/golden/digests/cfg5.tsv


def _worker(rank, world, port, out):
    import sys
    import torch.distributed as dist
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2208_09985_b200 as sg
    from paper_2208_09985_b200 import shard
    import oracle_ffi as O
    first, count = shard.rank_range(rank, world, 100000)
    gathered = [None] * world
    dist.all_gather_object(gathered, (first, count))
    t = shard.max_over_ranks(1.5 + rank)

    batch = sg.synth_packed(5, 0, N_CFG5)
    sh, pos, is_gathered = shard.plan(batch, world)
    mine = shard.members(sh, pos, rank)
    spec = O.baseline_spec(5)
    results = []
    for k in mine:
        tx, px = O.synth_pair(spec, int(k))
        a = O.align(tx, px, W=64, O=24)
        results.append((int(k), a.distance, a.windows, [a.counters[n] for n in O.COUNTER_NAMES],
                        a.cigar))
    parts = [None] * world
    dist.all_gather_object(parts, results)
    dist.barrier()
    if rank == 0:
        out.put((gathered, t, is_gathered, parts))
    dist.destroy_process_group()


def test_sharded_alignment_gloo():
    import golden_io as G
    import oracle_ffi as O
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 2000)
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    gathered, t, is_gathered, parts = q.get(timeout=600)
    for p in ps:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert gathered == [(0, 100000), (100000, 100000)]
    assert t == 2.5
    assert is_gathered  # cfg5's mix is bucketed, not split by input order
    assert all(len(p) > 0 for p in parts)
    rows = sorted((r for p in parts for r in p), key=lambda r: r[0])
    assert [r[0] for r in rows] == list(range(N_CFG5))  # every pair exactly once
    runs = [O.runs_from_cigar(r[4]) for r in rows]
    off = np.zeros(N_CFG5 + 1, np.int64)
    off[1:] = np.cumsum([len(x) for x in runs])
    got, _ = O.digest_blocks(np.array([r[1] for r in rows]), np.array([r[2] for r in rows]), None,
                             off, np.frombuffer(b"".join(runs), np.uint8),
                             np.array([r[3] for r in rows], np.uint64))
    blocks, *_ = G.read_digests("cfg5.tsv")
    assert got[0] == blocks[0][2]


@pytest.mark.parametrize("cfg_id,count,expect_gathered", [(5, 4000, True), (3, 400, False),
                                                          (2, 20000, False)])
def test_plan_shards_cover_and_balance(sg, cfg_id, count, expect_gathered):
    from paper_2208_09985_b200 import shard
    batch = sg.synth_packed(cfg_id, 0, count)
    tl, pl = batch.lengths()
    for parts in (1, 2, 4, 8):
        sh, pos, gathered = shard.plan(batch, parts)
        assert gathered == (expect_gathered and parts > 1)
        assert sh.min() >= 0 and sh.max() < parts
        lens = (tl + pl).astype(np.float64)
        loads = []
        for d in range(parts):
            mem = shard.members(sh, pos, d)
            assert sorted(pos[mem].tolist()) == list(range(len(mem)))  # a permutation
            if not gathered:  # contiguous ranges of input order
                assert (np.diff(mem) == 1).all()
            loads.append(lens[mem].sum())
        # the estimated cost weighs unrelated pairs more, so balance by length is loose
        assert max(loads) - min(loads) <= 5 * lens.max() + 0.1 * lens.sum() / parts
    with pytest.raises(sg.ConfigError):
        shard.plan(batch, 0)
    with pytest.raises(ValueError):
        shard.rank_range(2, 2, 10)
