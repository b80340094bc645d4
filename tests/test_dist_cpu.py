"""Data-parallel host logic on CPU: world_size-2 gloo process groups.

The N>1 path shards seed batches across ranks with no data-path collective
and all-reduces the flat gradient once per step.  These tests
run the same host functions the trainer uses (shard_plan, allreduce_mean)
in two real processes.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2110_08450_b200.prep import make_epoch_plan
from paper_2110_08450_b200.train import allreduce_mean, shard_plan


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n_ids, batch, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        plan = make_epoch_plan(np.arange(n_ids), batch, shuffle_seed=3)
        descs, host = shard_plan(plan, batch, rank, world)
        # every rank runs the same number of steps (zero-gradient padding)
        steps = torch.tensor([len(descs)])
        all_steps = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(all_steps, steps)
        got = [d[0] for d in descs.tolist() if d[0] >= 0]
        gathered = [None] * world
        dist.all_gather_object(gathered, got)
        # gradient averaging: rank-dependent flat gradients
        g = torch.arange(10, dtype=torch.float32) * (rank + 1)
        allreduce_mean(g, world)
        want = torch.arange(10, dtype=torch.float32) * (sum(range(1, world + 1)) / world)
        # seeds of this rank's batches come from the concatenated plan at the desc offsets
        perm = np.concatenate([b.dst_ids for b in plan.batches])
        ok_offsets = all(np.array_equal(perm[o:o + n], sb.dst_ids)
                         for (bid, o, n), sb in zip(descs.tolist(), host) if sb is not None)
        q.put((rank, [int(s) for s in all_steps], gathered, bool(torch.allclose(g, want)),
               ok_offsets, len(plan)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n_ids,batch", [(10_000, 1024), (8_192, 1024), (500, 64)])
def test_seed_sharding_and_gradient_mean_world2(n_ids, batch):
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_ids, batch, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, steps, gathered, grad_ok, off_ok, nb in res:
        assert len(set(steps)) == 1                     # lock-step ranks
        assert steps[0] == -(-nb // world)
        flat = [b for r in gathered for b in r]
        assert sorted(flat) == list(range(nb))          # every batch exactly once
        assert set(gathered[0]).isdisjoint(gathered[1])
        assert grad_ok and off_ok


def test_shard_plan_single_rank_is_identity():
    plan = make_epoch_plan(np.arange(1000), 128, 1)
    descs, host = shard_plan(plan, 128, 0, 1)
    assert [d[0] for d in descs.tolist()] == list(range(len(plan)))
    assert descs[-1, 2] == 1000 - 128 * 7


@pytest.mark.parametrize("n", [0, 1, 1023, 1024, 1025, 5000])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_chunk_descs_equals_shard_plan_of_chunked_ids(n, world):
    """Evaluator.set_ids builds its descriptors with chunk_descs (one sort, no
    SeedBatch per chunk): the same table shard_plan gives for the in-order chunks."""
    from paper_2110_08450_b200.prep import EpochPlan
    from paper_2110_08450_b200.sampler import SeedBatch
    from paper_2110_08450_b200.train import chunk_descs
    ids = np.random.default_rng(n).choice(10**7, n, replace=False).astype(np.int64)
    bs = 1024
    batches = tuple(SeedBatch(i, ids[s:s + bs]) for i, s in enumerate(range(0, n, bs)))
    plan = EpochPlan(batches=batches, batch_size=bs, shuffle_seed=0)
    for rank in range(world):
        want, _ = shard_plan(plan, bs, rank, world)
        got = chunk_descs(ids, bs, rank, world)
        assert got.shape == want.shape and (got == want).all()


def test_chunk_descs_rejects_duplicate_seeds_within_a_chunk():
    from paper_2110_08450_b200.train import chunk_descs
    ids = np.arange(3000)
    ids[10] = ids[1500]          # different chunks: allowed, as with SeedBatch
    chunk_descs(ids, 1024, 0, 1)
    ids[2500] = ids[2100]        # same (last, partial) chunk
    with pytest.raises(ValueError, match="seed IDs must be distinct"):
        chunk_descs(ids, 1024, 0, 1)
