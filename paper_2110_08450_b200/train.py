"""Data-parallel GraphSAGE training with on-device batch preparation.

The paper's training loop (PAPER.md:407-416 listing, 2562-2586 model) with
SALIENT's pipeline moved onto the GPU:

  prep stream   : sample MFG (sal_sample_mfg) -> gather features -> labels
                  for batch i+1, into device slot (i+1) % S
  compute stream: GraphSAGE fwd/bwd on slot i % S, gradient allreduce
                  (NCCL over NVLink when world > 1), fused Adam

Shapes are static: every layer is padded to the plan's worst-case
destination count (node_cap) and kernels read the true counts from device
memory, so a step needs no host synchronisation and can be captured in a
CUDA graph (`graphs=True`).  Seed nodes are sharded across ranks: global
step s of an epoch trains plan batch s*W + r on rank r (effective batch
1024*W); a rank without a batch in the last step
contributes a zero gradient.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch
import torch.nn.functional as F

from . import _lib
from .graph import DeviceGraph
from .model import GraphSAGE
from .prep import gather_rows, make_epoch_plan
from .sampler import FanoutSpec, MfgWorkspace, RNG_POLICIES


@dataclass
class TrainConfig:
    fanouts: FanoutSpec = field(default_factory=lambda: FanoutSpec((15, 10, 5)))
    batch_size: int = 1024
    hidden: int = 256
    lr: float = 0.003
    dropout: float = 0.5
    act_dtype: torch.dtype = torch.bfloat16
    global_seed: int = 1
    shuffle_seed: int = 1
    depth: int = 1                 # batches prepared ahead of the consumer
    gather_free: bool = False      # layer-0 mean straight from the feature table
    rng_policy: str = "splitmix"
    graphs: bool = False           # capture prep+step in CUDA graphs


class _Slot:
    def __init__(self, dg: DeviceGraph, cfg: TrainConfig, device):
        self.ws = MfgWorkspace(dg.num_nodes, cfg.fanouts, cfg.batch_size, device=device)
        rows = self.ws.node_cap[-1] if not cfg.gather_free else self.ws.node_cap[-2]
        f = dg.features.shape[1]
        self.feats = torch.zeros((max(rows, 1), f), dtype=dg.features.dtype, device=device)
        self.labels = torch.full((cfg.batch_size,), -1, dtype=torch.int64, device=device)
        self.desc = torch.zeros(3, dtype=torch.int64, device=device)
        self.seeds = torch.zeros(cfg.batch_size, dtype=torch.int64, device=device)
        self.done = torch.cuda.Event()
        self.free = torch.cuda.Event()


class Trainer:
    """One rank of the data-parallel trainer."""

    def __init__(self, dg: DeviceGraph, train_ids: np.ndarray, cfg: TrainConfig = TrainConfig(),
                 rank: int = 0, world: int = 1, num_classes: int | None = None):
        _lib.require_cuda()
        if dg.features is None or dg.labels is None:
            raise ValueError("trainer needs a DeviceGraph with features and labels")
        self.dg, self.cfg = dg, cfg
        self.rank, self.world = rank, world
        self.device = dg.device
        self.train_ids = np.asarray(train_ids, dtype=np.int64)
        self.num_classes = num_classes or dg.num_classes
        self.nh = len(cfg.fanouts)
        torch.manual_seed(cfg.global_seed)
        self.model = GraphSAGE(dg.num_features, cfg.hidden, self.num_classes, self.nh,
                               cfg.dropout).to(self.device)
        params = list(self.model.parameters())
        total = sum(p.numel() for p in params)
        self.flat_grad = torch.zeros(total, dtype=torch.float32, device=self.device)
        off = 0
        for p in params:
            p.grad = self.flat_grad[off:off + p.numel()].view_as(p)
            off += p.numel()
        self.opt = torch.optim.Adam(params, lr=cfg.lr, fused=True)
        self.slots = [_Slot(dg, cfg, self.device) for _ in range(cfg.depth + 1)]
        self.prep_stream = torch.cuda.Stream(device=self.device)
        self.policy = RNG_POLICIES[cfg.rng_policy]
        self.x_table = dg.feature_view()
        self.loss_sum = torch.zeros((), dtype=torch.float32, device=self.device)
        self.epoch = -1
        self.steps_per_epoch = 0

    # ---------------------------------------------------------------- plan
    def set_epoch(self, epoch: int) -> int:
        """Shuffle (make_epoch_plan with shuffle_seed + epoch), shard, upload."""
        plan = make_epoch_plan(self.train_ids, self.cfg.batch_size, self.cfg.shuffle_seed + epoch)
        nb = len(plan)
        W, r = self.world, self.rank
        self.steps_per_epoch = math.ceil(nb / W) if nb else 0
        self.host_batches = []
        descs = []
        for s in range(self.steps_per_epoch):
            b = s * W + r
            if b < nb:
                sb = plan.batches[b]
                descs.append((sb.batch_id, b * self.cfg.batch_size, len(sb)))
                self.host_batches.append(sb)
            else:
                descs.append((-1, 0, 0))
                self.host_batches.append(None)
        perm = np.concatenate([b.dst_ids for b in plan.batches]) if nb else np.zeros(1, np.int64)
        self.seeds_all = torch.from_numpy(perm).to(self.device)
        self.desc_all = torch.from_numpy(np.asarray(descs, dtype=np.int64).reshape(-1, 3)).to(
            self.device)
        self.seeds_pinned = torch.from_numpy(perm).pin_memory()
        self.desc_pinned = torch.from_numpy(np.asarray(descs, dtype=np.int64).reshape(-1, 3)
                                            ).pin_memory()
        self.epoch = epoch
        self.plan = plan
        return self.steps_per_epoch

    # ---------------------------------------------------------------- prep
    def _enqueue_prep(self, slot: _Slot, step: int, host_inputs: bool = False) -> None:
        ws = slot.ws
        st = self.prep_stream
        with torch.cuda.stream(st):
            st.wait_event(slot.free)
            if host_inputs:
                # end-to-end mode: this step's seeds + descriptor come from pinned host memory
                d = self.desc_pinned[step]
                n = int(d[2])
                slot.desc.copy_(d, non_blocking=True)
                if n:
                    off = int(d[1])
                    slot.seeds[:n].copy_(self.seeds_pinned[off:off + n], non_blocking=True)
                slot.desc[1:2].zero_()
                seeds_base, desc = slot.seeds, slot.desc
            else:
                seeds_base, desc = self.seeds_all, self.desc_all[step]
            ws.run(self.dg, seeds_base, desc, self.cfg.global_seed, self.policy, st)
            L = self.nh
            rows = ws.node_cap[L] if not self.cfg.gather_free else ws.node_cap[L - 1]
            n_dev = ws.sizes[L:L + 1] if not self.cfg.gather_free else ws.sizes[L - 1:L]
            gather_rows(self.x_table, ws.globals, slot.feats[:, :self.x_table.shape[1]],
                        n=rows, n_dev=n_dev, stream=st)
            _lib.check(_lib.lib().sal_gather_labels(
                self.dg.labels.data_ptr(), seeds_base.data_ptr(), desc.data_ptr(),
                self.cfg.batch_size, slot.labels.data_ptr(), _lib.stream_ptr(st)),
                "gather_labels")
            slot.done.record(st)

    # ---------------------------------------------------------------- step
    def _adjs(self, slot: _Slot):
        ws = slot.ws
        L = self.nh
        out = []
        for i in range(L):
            h = L - 1 - i
            out.append((ws.dst_indptr[h], ws.src_local[h], ws.node_cap[h], ws.sizes[h:h + 1]))
        return out

    def _step_compute(self, slot: _Slot) -> torch.Tensor:
        cs = torch.cuda.current_stream()
        cs.wait_event(slot.done)
        self.flat_grad.zero_()
        x_global = (self.x_table, slot.ws.globals) if self.cfg.gather_free else None
        out = self.model(slot.feats, self._adjs(slot), self.cfg.act_dtype, x_global=x_global)
        nll = F.nll_loss(out, slot.labels, ignore_index=-1, reduction="sum")
        cnt = (slot.labels >= 0).sum().clamp_min(1).to(torch.float32)
        loss = nll / cnt
        loss.backward()
        if self.world > 1:
            torch.distributed.all_reduce(self.flat_grad, op=torch.distributed.ReduceOp.AVG)
        self.opt.step()
        slot.free.record(cs)
        return loss.detach()

    def train_steps(self, start: int, count: int, host_inputs: bool = False,
                    loss_out: torch.Tensor | None = None) -> torch.Tensor:
        """Run steps [start, start+count) of the current epoch; returns the
        device tensor of per-step losses.  With host_inputs, seeds come from
        pinned host memory each step and every loss is copied back to
        `loss_out` (pinned) — the end-to-end path."""
        self.model.train()
        S = len(self.slots)
        losses = torch.zeros(count, dtype=torch.float32, device=self.device)
        depth = self.cfg.depth
        for k in range(min(depth, count)):
            self._enqueue_prep(self.slots[(start + k) % S], start + k, host_inputs)
        for k in range(count):
            step = start + k
            if k + depth < count:
                self._enqueue_prep(self.slots[(step + depth) % S], step + depth, host_inputs)
            loss = self._step_compute(self.slots[step % S])
            losses[k] = loss
            if loss_out is not None:
                loss_out[k].copy_(loss, non_blocking=True)
        return losses

    def train_epoch(self, epoch: int) -> float:
        n = self.set_epoch(epoch)
        losses = self.train_steps(0, n)
        return float(losses.mean().item()) if n else 0.0

    # ---------------------------------------------------------------- eval
    @torch.no_grad()
    def evaluate(self, ids: np.ndarray, fanouts: FanoutSpec | None = None,
                 batch_size: int | None = None) -> tuple[int, int]:
        """Sampled inference over `ids` (this rank's shard); returns (correct, total)."""
        from .prep import PrepConfig, run_epoch_prep
        from .prep import EpochPlan
        from .sampler import SeedBatch
        self.model.eval()
        fan = fanouts or self.cfg.fanouts
        bs = batch_size or self.cfg.batch_size
        ids = np.asarray(ids, dtype=np.int64)
        batches = tuple(SeedBatch(i, ids[s:s + bs]) for i, s in enumerate(range(0, len(ids), bs)))
        plan = EpochPlan(batches=batches, batch_size=bs, shuffle_seed=0)
        correct = torch.zeros((), dtype=torch.int64, device=self.device)
        total = 0
        x = self.dg.feature_view()
        cfg = PrepConfig(num_workers=2, fanouts=fan, feature_dtype="f16"
                         if x.dtype == torch.float16 else "f32")
        for pb in run_epoch_prep(self.dg, x, self.dg.labels, plan, cfg, self.cfg.global_seed + 7):
            adjs = [(l.indptr, l.src_local, l.num_dst, None) for l in pb.mfg.layers]
            out = self.model(pb.features, adjs, self.cfg.act_dtype)
            correct += (out.argmax(dim=-1) == pb.labels).sum()
            total += len(pb.labels)
        self.model.train()
        return int(correct.item()), total
