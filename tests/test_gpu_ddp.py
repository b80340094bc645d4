"""Data-parallel training step on one GPU: two gloo ranks sharing cuda:0.

* The averaged gradient of a W=2 step equals the mean of the two W=1 gradients of
  the same plan batches (reference: PAPER.md:1702-1717, DDP over seed shards;
  lr = 0 keeps the weights at their initial values for the W=1 comparator).
* A W=2 epoch whose last step gives rank 1 an empty batch (shard_plan pads with
  batch_id -1) keeps gradients and parameters finite on every rank, with the
  caching allocator pre-filled with NaN so any read of unwritten padding rows shows.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

N, F, C, BATCH = 20_000, 128, 16, 256


def _graph():
    from paper_2110_08450_b200.graph import synth_graph_device
    return synth_graph_device(N, 12.0, 3.0, seed=4, num_features=F, num_classes=C,
                              feature_seed=4, label_seed=4)


def _nan_fill_allocator():
    """Leave NaN bytes in the caching allocator's free blocks."""
    blocks = [torch.full((1 << 24,), float("nan"), device="cuda") for _ in range(8)]
    del blocks


def _trainer(dg, train, rank, world, graphs):
    from paper_2110_08450_b200.train import TrainConfig, Trainer
    cfg = TrainConfig(batch_size=BATCH, dropout=0.0, lr=0.0, gather_free=True, graphs=graphs)
    return Trainer(dg, train, cfg, rank=rank, world=world)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    torch.distributed.init_process_group("gloo", rank=rank, world_size=world)
    try:
        dg = _graph()
        train = np.arange(0, N, 7)
        tr = _trainer(dg, train, rank, world, graphs=False)
        tr.set_epoch(0)
        tr.begin_epoch()
        tr.run_steps(0, 1)
        torch.cuda.synchronize()
        g = tr.model.grad.cpu().numpy()
        # a short epoch whose last step is empty on rank 1: 3 plan batches, 2 steps
        _nan_fill_allocator()
        tr2 = _trainer(dg, np.arange(0, 3 * BATCH - 17), rank, world, graphs=True)
        tr2.model.lr = 0.01
        steps = tr2.set_epoch(0)
        tr2.begin_epoch()
        finite = []
        for k in range(steps):
            tr2.run_steps(k, 1)
            torch.cuda.synchronize()
            finite.append(bool(torch.isfinite(tr2.model.grad).all())
                          and bool(torch.isfinite(tr2.model.flat).all()))
        q.put((rank, g, steps, finite, tr2.desc_host.tolist()))
    finally:
        torch.distributed.destroy_process_group()


def test_ddp_gradient_equals_single_rank_mean_and_empty_batch_is_finite():
    # W = 1 comparator: plan batches 0 and 1 at the initial weights (lr = 0)
    dg = _graph()
    train = np.arange(0, N, 7)
    tr = _trainer(dg, train, 0, 1, graphs=False)
    tr.set_epoch(0)
    tr.begin_epoch()
    tr.run_steps(0, 1)
    torch.cuda.synchronize()
    g0 = tr.model.grad.clone()
    tr.run_steps(1, 1)
    torch.cuda.synchronize()
    g1 = tr.model.grad.clone()
    want = ((g0 + g1) / 2).cpu().numpy()
    del tr, dg
    torch.cuda.empty_cache()

    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=600) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    scale = np.abs(want).max()
    for rank, g, steps, finite, descs in res:
        # split-K weight-gradient atomics and the reverse adjacency make the fp32
        # summation order nondeterministic: tolerance, not bits
        assert np.allclose(g, want, rtol=1e-3, atol=1e-4 * scale), (rank, np.abs(g - want).max())
        assert steps == 2
        assert all(finite), (rank, finite)
    assert res[1][4][1][0] == -1          # rank 1's last step is the empty padding batch
