"""Data-parallel GraphSAGE training with on-device batch preparation.

The paper's training loop (PAPER.md:407-416 listing, 2562-2586 model) with
SALIENT's pipeline moved onto the GPU:

  prep stream   : plan cursor -> sample MFG (sal_sample_mfg) -> destination
                  feature rows (fp16 table -> bf16), for batch i+1, into device
                  slot (i+1) % 2
  late stream   : labels + reverse adjacency of batch i (+ zeroing of the
                  tcgen05 gradient blocks), beside batch i's forward pass
  compute stream: GraphSAGE fwd/bwd on slot i % 2 (FusedSAGE; layer 0 reads its
                  sampled rows straight from the table when gather_free), weight
                  gradients of the upper layers on a side stream, gradient
                  all-reduce (NCCL over NVLink when world > 1), fused Adam

Shapes are static: each layer is padded to the plan's worst-case destination
count (node_cap) and the kernels read the true counts from device memory, so
a step has no host synchronisation.  With `graphs=True` the pair
{prep(i+1) || train(i)} is captured once per slot parity and replayed; the
device epoch cursor (sal_plan_next) makes every replay prepare the next batch
of the plan.  Seed nodes are sharded across ranks: step s trains plan batch
s*W + r on rank r (effective batch 1024*W); a rank
without a batch in the last step contributes a zero gradient.  The
end-to-end mode (host_inputs) feeds each step's seeds from pinned host memory
and reads each loss back (Trainer.run_steps).  Evaluator runs sampled
inference on the same machinery.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .graph import DeviceGraph
from .model import FusedSAGE, build_transpose
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
    gather_free: bool = False      # layer-0 mean straight from the feature table
    rng_policy: str = "splitmix"
    graphs: bool = True            # capture {prep || step} in CUDA graphs
    model_seed: int = 0
    prep_priority: int = 0         # CUDA stream priority of the prep stream (lower = higher)
    late_priority: int = 0         # ... of the stream building labels / reverse adjacency
    compute_priority: int = 0      # ... of the training stream (0: the caller's stream)
    wgrad_priority: int = 0        # ... of the model's overlapped weight-gradient stream
    tc_wgrad: bool = True          # tcgen05 weight gradients where the shapes allow
    wgrad_fork_late: bool = True   # overlapped weight gradients fork after the dA GEMM
    late_prep: bool = True         # labels + reverse adjacency built beside the forward pass
    sampler_lanes: int = 0         # lanes per destination (0 = smallest group holding the fanout)
    sampler_bps: int = 0           # sampler grid cap in blocks per SM (0 = 8)
    table_factor: int = 1          # id-table capacity multiplier (lower load, fewer probes)
    # gather_free: the last hop sampled straight into the layer-0 mean + self rows by one
    # kernel (sal_sample_aggregate) instead of sample -> src_glob -> mean + row gather
    fuse_last_hop: bool = True
    fused_on_prep: bool = True     # ... on the prep stream (False: first kernel of the step)
    # resident blocks per SM of the fused last hop in training: three 4-warp blocks leave
    # room for a 3-stage tcgen05 weight-gradient CTA beside them (164 -> 161 us per step)
    fused_bps: int = 3
    # hop L-2's resolve inside the fused kernel (sal_mfg_plan.resolve_in_aggregate)
    fused_resolve: bool = True


def shard_plan(plan, batch_size: int, rank: int, world: int):
    """Seed-node sharding of one epoch: global step s trains plan
    batch s*world + rank on this rank; ranks past the end of the plan get an
    empty batch (batch_id -1) and contribute a zero gradient.

    Returns (descs int64 [steps, 3] = (batch_id, seed_offset, n_seeds) into the
    concatenated plan, host SeedBatch or None per step)."""
    nb = len(plan)
    steps = math.ceil(nb / world) if nb else 0
    descs = np.zeros((steps, 3), dtype=np.int64)
    host = []
    for s in range(steps):
        b = s * world + rank
        if b < nb:
            sb = plan.batches[b]
            descs[s] = (sb.batch_id, b * batch_size, len(sb))
            host.append(sb)
        else:
            descs[s] = (-1, 0, 0)
            host.append(None)
    return descs, host


def check_chunks_distinct(ids: np.ndarray, batch_size: int) -> None:
    """The distinct-seeds check of a SeedBatch (sampler.py) for every in-order chunk of
    `ids`, in one sort."""
    n = len(ids)
    nf = n // batch_size
    full = np.sort(ids[:nf * batch_size].reshape(nf, batch_size), axis=1)
    tail = np.sort(ids[nf * batch_size:])
    if (full[:, 1:] == full[:, :-1]).any() or (tail[1:] == tail[:-1]).any():
        raise ValueError("seed IDs must be distinct")


def chunk_descs(ids: np.ndarray, batch_size: int, rank: int, world: int,
                check: bool = True) -> np.ndarray:
    """shard_plan of `ids` chunked in order (batch_id = chunk index), without building
    a SeedBatch per chunk: the same descriptors (and, with `check`, the same
    distinct-seeds check)."""
    n = len(ids)
    nb = -(-n // batch_size) if n else 0
    if check:
        check_chunks_distinct(ids, batch_size)
    steps = -(-nb // world) if nb else 0
    b = np.arange(steps, dtype=np.int64) * world + rank
    live = b < nb
    descs = np.zeros((steps, 3), dtype=np.int64)
    descs[:, 0] = np.where(live, b, -1)
    descs[:, 1] = np.where(live, b * batch_size, 0)
    descs[:, 2] = np.where(live, np.minimum(batch_size, n - b * batch_size), 0)
    return descs


def allreduce_mean(t: torch.Tensor, world: int) -> None:
    """In-place mean over ranks: NCCL AVG (NVLink/NVLS), SUM / world elsewhere."""
    if world <= 1:
        return
    backend = torch.distributed.get_backend()
    if backend == "nccl":
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.AVG)
    else:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.SUM)
        t.div_(world)


def _model_width(dg: DeviceGraph) -> int:
    """Feature width the model consumes: at least the table's padded row (16-byte
    multiple), so every layer-0 row is whole 16-byte vectors for the fast kernels,
    and 128 for 16-bit tables between 64 and 128 columns, so layer 0 runs on the
    tcgen05 kernels (K = 2 x 128).  Products' 100 fp16 columns: the table is stored at
    128 already (graph._pad_cols), so is the model.  The padding columns are zero and their weights get zero gradient, so
    the model is the unpadded one."""
    fp = dg.features.shape[1]
    if dg.features.element_size() == 2 and 64 < fp < 128:
        return 128
    return fp


def philox_epoch_seed(global_seed: int, epoch: int) -> int:
    """The Philox key of one training epoch: splitmix64 of (global_seed, epoch)."""
    from .sampler import MASK64, _fmix
    return _fmix((global_seed ^ _fmix((epoch + 0x9E3779B97F4A7C15) & MASK64)) & MASK64)


def _fusable(dg: DeviceGraph, cfg: TrainConfig) -> bool:
    """sal_sample_aggregate's shape limits: fp16 table rows of 16-byte multiples up to
    256 bytes, last-hop fanout <= 32, 16-bit activations."""
    x = dg.features
    return (cfg.gather_free and cfg.fuse_last_hop and x.dtype == torch.float16
            and (x.shape[1] * 2) % 16 == 0 and x.shape[1] * 2 <= 256
            and (x.stride(0) * 2) % 16 == 0 and cfg.fanouts.per_hop[0] <= 32
            and cfg.act_dtype in (torch.bfloat16, torch.float16))


def _model_table(dg: DeviceGraph) -> torch.Tensor:
    f, fp = dg.num_features, dg.features.shape[1]
    if fp != f:
        dg.features[:, f:].zero_()
    return dg.features


class _Slot:
    def __init__(self, dg: DeviceGraph, cfg: TrainConfig, device, backward: bool = True):
        # gather-free: layer 0 reads rows by global id, so the last hop needs no relabel
        self.fused = _fusable(dg, cfg)
        self.ws = MfgWorkspace(dg.num_nodes, cfg.fanouts, cfg.batch_size, device=device,
                               last_hop_edges=cfg.gather_free, sample_lanes=cfg.sampler_lanes,
                               sample_bps=cfg.sampler_bps, table_factor=cfg.table_factor,
                               last_hop_fused=self.fused,
                               aggregate_bps=cfg.fused_bps if backward else 0,
                               reset_in_aggregate=True,
                               # hop L-2's resolve inside the fused kernel: sampled inference
                               # 0.0543 -> 0.0528 s, the training step 147.5 -> 146.0 us
                               resolve_in_aggregate=(not backward) or cfg.fused_resolve)
        ws = self.ws
        nh = ws.num_hops
        rows = ws.node_cap[-1] if not cfg.gather_free else ws.node_cap[-2]
        f = _model_width(dg)
        # layer-0 "cat" buffer: right half = gathered features, left = mean
        self.feats = torch.zeros((max(rows, 1), 2 * f), dtype=cfg.act_dtype, device=device)
        self.labels = torch.full((cfg.batch_size,), -1, dtype=torch.int64, device=device)
        self.desc = torch.zeros(3, dtype=torch.int64, device=device)
        self.seeds = torch.zeros(max(cfg.batch_size, 1), dtype=torch.int64, device=device)
        self.desc_used = self.desc   # the descriptor the last prep read (fused last hop)
        # late-stream milestones: labels + zeroed gradient blocks, reverse adjacency of layer i
        self.ev_head = torch.cuda.Event()
        self.ev_t = [torch.cuda.Event() for _ in range(ws.num_hops)]
        # reverse adjacency of layers i >= 1 (hop h = L-1-i), built on the prep stream
        L = _lib.lib()
        self.transposes = [None]
        self.t_ws = [None]
        for i in range(1, nh if backward else 1):
            h = nh - 1 - i
            n_src = ws.node_cap[h + 1]
            self.transposes.append((
                torch.zeros(n_src + 1, dtype=torch.int32, device=device),
                torch.zeros(max(ws.edge_cap[h], 1), dtype=torch.int32, device=device),
                torch.zeros(max(ws.edge_cap[h], 1), dtype=torch.float32, device=device)))
            nb = -(-L.sal_transpose_ws_bytes(n_src) // 16) * 16   # 16 B multiple (zero_spans)
            tws = torch.empty(nb, dtype=torch.uint8, device=device)
            self.t_ws.append(tws)
            # the build also lists the rows the input gradient handles source-major
            lo, co = ctypes.c_int64(), ctypes.c_int64()
            _lib.check(L.sal_transpose_complex_list(n_src, ctypes.byref(lo), ctypes.byref(co)),
                       "transpose_complex_list")
            self.transposes[-1] = self.transposes[-1] + (
                tws[lo.value:lo.value + 4 * max(n_src, 1)].view(torch.int32),
                tws[co.value:co.value + 4].view(torch.int32))


class _Staging:
    """One step's host inputs for the end-to-end path: [desc(3) | seeds] in pinned
    memory, copied H2D as one block into a device mirror that the captured step
    graphs read (no memcpy node inside the graph)."""

    def __init__(self, batch_size: int, device):
        self.host = torch.zeros(3 + max(batch_size, 1), dtype=torch.int64).pin_memory()
        self.np = self.host.numpy()
        self.dev = torch.zeros(3 + max(batch_size, 1), dtype=torch.int64, device=device)
        self.ddesc = self.dev[:3]
        self.dseeds = self.dev[3:]
        self.ev = torch.cuda.Event()       # the last replay that read `dev` has finished
        self.copied = torch.cuda.Event()   # `dev` holds this step's inputs


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
        self.model = FusedSAGE(_model_width(dg), cfg.hidden, self.num_classes, self.nh,
                               cfg.dropout, device=self.device, seed=cfg.model_seed,
                               act_dtype=cfg.act_dtype, lr=cfg.lr)
        self.model.tc_wgrad = cfg.tc_wgrad
        self.model.wgrad_fork_late = cfg.wgrad_fork_late
        if cfg.wgrad_priority != 0:
            self.model._wgrad_stream = torch.cuda.Stream(device=self.device,
                                                         priority=cfg.wgrad_priority)
        if world > 1:  # identical initial weights on every rank
            torch.distributed.broadcast(self.model.flat, src=0)
            self.model.refresh_shadow()
        self.loss_buf = torch.zeros((), dtype=torch.float32, device=self.device)
        # pipeline depth: batches in flight (one trained, one prepared).  Three slots with
        # {hops(k+2) || fused fill(k+1) || train(k)} trained the same batches and measured
        # 171 against 148 us per step (the fill then contends with the forward): not kept
        self.depth = 2
        self.slots = [_Slot(dg, cfg, self.device) for _ in range(self.depth)]
        self.ring = 2 * self.depth   # pinned staging buffers of the end-to-end path
        self.staging = [_Staging(cfg.batch_size, self.device) for _ in range(self.ring)]
        self.copy_stream = torch.cuda.Stream(device=self.device)
        self._loss_ev = [torch.cuda.Event() for _ in range(8)]
        # high priority: the prep chain is latency-bound (many small dependent kernels), so
        # it should take SMs first as the bandwidth-bound training kernels drain
        self.prep_stream = torch.cuda.Stream(device=self.device, priority=cfg.prep_priority)
        # the backward-only inputs of the step being trained (labels, reverse adjacency)
        # are built on a third stream while its forward pass runs
        self.late_stream = torch.cuda.Stream(device=self.device, priority=cfg.late_priority)
        # optional dedicated training stream (priority != 0); run_steps joins it back to
        # the caller's stream, so events the caller records stay valid
        self.compute_stream = (torch.cuda.Stream(device=self.device, priority=cfg.compute_priority)
                               if cfg.compute_priority != 0 else None)
        self.policy = RNG_POLICIES[cfg.rng_policy]
        self.sample_seed = cfg.global_seed
        self.x_table = _model_table(dg)
        self.cursor = torch.zeros(1, dtype=torch.int64, device=self.device)
        self.step_ctr = torch.zeros(1, dtype=torch.int64, device=self.device)
        self.losses = torch.zeros(1, dtype=torch.float32, device=self.device)
        self.last_loss = torch.zeros((), dtype=torch.float32, device=self.device)
        self.ticket = torch.zeros(1, dtype=torch.int32, device=self.device)   # adam_step_tail
        self.graphs = {}
        self.graph_kernels = {}
        self.graph_allreduce = True    # NCCL all-reduce captured inside the step graph
        self.kernel_launches = 0   # library kernels executed by run_steps (launch audit)
        self.steps_per_epoch = 0
        self.seeds_all = torch.zeros(1, dtype=torch.int64, device=self.device)
        self.desc_all = torch.zeros((1, 3), dtype=torch.int64, device=self.device)

    # ---------------------------------------------------------------- plan
    def set_epoch(self, epoch: int) -> int:
        """Shuffle (make_epoch_plan with shuffle_seed + epoch), shard, upload."""
        plan = make_epoch_plan(self.train_ids, self.cfg.batch_size, self.cfg.shuffle_seed + epoch)
        nb = len(plan)
        descs, self.host_batches = shard_plan(plan, self.cfg.batch_size, self.rank, self.world)
        self.steps_per_epoch = len(descs)
        descs = [tuple(d) for d in descs]
        perm = np.concatenate([b.dst_ids for b in plan.batches]) if nb else np.zeros(1, np.int64)
        # copy into persistent buffers (captured graphs hold their addresses)
        if self.seeds_all.numel() < len(perm):
            self.seeds_all = torch.zeros(len(perm), dtype=torch.int64, device=self.device)
            self.graphs.clear()
        if self.desc_all.shape[0] < max(1, len(descs)):
            self.desc_all = torch.zeros((max(1, len(descs)), 3), dtype=torch.int64,
                                        device=self.device)
            self.losses = torch.zeros(max(1, len(descs)), dtype=torch.float32,
                                      device=self.device)
            self.graphs.clear()
        self.seeds_all[:len(perm)].copy_(torch.from_numpy(perm))
        if descs:
            self.desc_all[:len(descs)].copy_(torch.from_numpy(np.asarray(descs, np.int64)))
        if getattr(self, "n_steps_dev", None) != len(descs):
            self.graphs.clear()  # the step count is baked into the captured plan_next
        self.n_steps_dev = len(descs)
        self.desc_host = np.asarray(descs, dtype=np.int64).reshape(-1, 3)
        self.perm_host = perm
        self.epoch = epoch
        self.plan = plan
        if self.cfg.rng_policy == "philox":
            # Philox streams are keyed on (seed, epoch) x (draw, node, hop, batch): a new
            # key each epoch (the graphs hold it by value, so they are re-captured);
            # splitmix keeps the reference's (global_seed, batch_id, hop) keying
            seed = philox_epoch_seed(self.cfg.global_seed, epoch)
            if seed != self.sample_seed:
                self.sample_seed = seed
                self.graphs.clear()
        self.cursor.zero_()
        self.step_ctr.zero_()
        return self.steps_per_epoch

    # ---------------------------------------------------------------- prep
    def _prep(self, slot: _Slot, stage: "_Staging | None", late: bool = False) -> None:
        """Enqueue one batch preparation on the current stream (capturable): seeds ->
        MFG -> layer-0 feature rows, plus (late=True) what _prep_late builds."""
        self._hops(slot, stage)
        self._fill(slot)
        if late:
            self._prep_late(slot, stage)

    def _hops(self, slot: _Slot, stage: "_Staging | None") -> None:
        """Plan cursor (or the staged H2D inputs) -> the slot's MFG (a fused last hop
        is left to _fill)."""
        ws = slot.ws
        st = torch.cuda.current_stream()
        if stage is not None:  # this step's inputs, already copied H2D (run_steps)
            desc, seeds_base = stage.ddesc, stage.dseeds
            ws.run(self.dg, seeds_base, desc, self.sample_seed, self.policy, st)
        else:  # the plan cursor's next step, advanced inside the first sampling kernel
            # (sal_sample_mfg_next: 147.2 -> 145.3 us per step against sal_plan_next + run)
            desc = slot.desc
            ws.run_next(self.dg, self.seeds_all, self.desc_all, self.n_steps_dev, self.cursor,
                        desc, self.sample_seed, self.policy, st)
        slot.desc_used = desc

    def _fill(self, slot: _Slot) -> None:
        """The slot's layer-0 input: the fused last hop, or the destination rows."""
        ws = slot.ws
        st = torch.cuda.current_stream()
        desc = slot.desc_used
        nh = self.nh
        f, fx = self.model.dims[0], self.x_table.shape[1]
        if slot.fused:
            if self.cfg.fused_on_prep:  # last hop -> layer-0 [mean | self] in one pass
                ws.aggregate(self.dg, self.x_table, slot.feats, f, desc, self.sample_seed,
                             self.policy, st)
        else:
            rows = ws.node_cap[nh] if not self.cfg.gather_free else ws.node_cap[nh - 1]
            n_dev = ws.sizes[nh:nh + 1] if not self.cfg.gather_free else ws.sizes[nh - 1:nh]
            gather_rows(self.x_table, ws.globals, slot.feats[:, f:f + fx], n=rows, n_dev=n_dev,
                        stream=st)

    def _prep_late(self, slot: _Slot, stage: "_Staging | None", zero_grads: bool = False) -> None:
        """The inputs only the loss / backward read: labels and the reverse adjacency
        of layers >= 1 (capturable, current stream); zero_grads: also clear the
        tcgen05 weight-gradient blocks of the step being trained."""
        ws = slot.ws
        st = torch.cuda.current_stream()
        L = _lib.lib()
        nh = self.nh
        seeds_base = stage.dseeds if stage is not None else self.seeds_all
        desc = stage.ddesc if stage is not None else slot.desc
        # every layer's count/scan workspace and (zero_grads) the tcgen05 gradient blocks
        # are zeroed by one kernel (no memset nodes in the captured chain)
        spans = [(t.data_ptr(), t.numel()) for t in slot.t_ws[1:]]
        if zero_grads:
            spans += self.model.tc_grad_spans()
        for c in range(0, len(spans), 8):   # sal_zero_spans takes up to 8 ranges per launch
            chunk = spans[c:c + 8]
            ptrs = (ctypes.c_void_p * len(chunk))(*[p for p, _ in chunk])
            nbytes = (ctypes.c_int64 * len(chunk))(*[b for _, b in chunk])
            _lib.check(L.sal_zero_spans(ptrs, nbytes, len(chunk), _lib.stream_ptr(st)),
                       "zero_spans")
        _lib.check(L.sal_gather_labels(self.dg.labels.data_ptr(), seeds_base.data_ptr(),
                                       desc.data_ptr(), self.cfg.batch_size,
                                       slot.labels.data_ptr(), _lib.stream_ptr(st)),
                   "gather_labels")
        # the output layer waits only for its labels and zeroed gradient block; each
        # layer's input gradient waits only for its own reverse adjacency, built in the
        # order the backward consumes them
        slot.ev_head.record(st)
        for i in reversed(range(1, nh)):
            h = nh - 1 - i
            build_transpose(ws.dst_indptr[h], ws.src_local[h], ws.sizes[h:h + 1], ws.node_cap[h],
                            ws.node_cap[h + 1], out=slot.transposes[i], ws=slot.t_ws[i],
                            ws_zeroed=True)
            slot.ev_t[i].record(st)

    def _adjs(self, slot: _Slot):
        ws = slot.ws
        out = []
        for i in range(self.nh):
            h = self.nh - 1 - i
            out.append((ws.dst_indptr[h], ws.src_local[h], ws.node_cap[h], ws.sizes[h:h + 1]))
        return out

    def _train(self, slot: _Slot, part: str = "all", late=None) -> None:
        """fwd + bwd [+ all-reduce] [+ Adam] on the current stream (capturable).

        part: "all" (one graph, the gradient all-reduce captured with it),
        "pre" (fwd + bwd only) or "post" (Adam + bookkeeping) — the split used
        when NCCL cannot be captured, with the all-reduce issued eagerly in
        between.  late: the stream building this slot's labels / reverse adjacency,
        joined after the forward pass."""
        m = self.model
        if part in ("all", "pre"):
            xg = (self.x_table, slot.ws.src_glob) if self.cfg.gather_free else None
            if slot.fused:
                xg = None
                if not self.cfg.fused_on_prep:
                    slot.ws.aggregate(self.dg, self.x_table, slot.feats, m.dims[0],
                                      slot.desc_used, self.sample_seed, self.policy,
                                      torch.cuda.current_stream())
            head = m.head_ok()
            logits, saved = m.forward(slot.feats, self._adjs(slot), x_global=xg,
                                      salt=m.t, head=head, mean0_ready=slot.fused)
            t_events = None
            if late is not None:   # wait for each late-stream input where it is consumed
                torch.cuda.current_stream().wait_event(slot.ev_head)
                t_events = slot.ev_t
            if head:  # output layer + loss on tcgen05, then the backward of every layer
                m.loss_backward(saved, slot.labels, self.loss_buf, slot.transposes,
                                grads_zeroed=late is not None, loss_zeroed=True,
                                t_events=t_events)
            else:
                loss, dlog = m.loss(logits, slot.labels, out=self.loss_buf, zeroed=True)
                m.backward(dlog, saved, slot.transposes, grads_zeroed=late is not None,
                           t_events=t_events)
            if late is not None:
                torch.cuda.current_stream().wait_stream(late)
        if part == "all" and self.world > 1:
            allreduce_mean(m.grad, self.world)
        if part in ("all", "post"):
            if m.act == torch.bfloat16 and m.flat.numel() % 4 == 0:
                # Adam + the per-step bookkeeping in one launch
                _lib.check(_lib.lib().sal_adam_step_tail(
                    m.flat.data_ptr(), m.grad.data_ptr(), m.m.data_ptr(), m.v.data_ptr(),
                    m.shadow.data_ptr(), m.flat.numel(), m.lr, m.betas[0], m.betas[1], m.eps,
                    m.t.data_ptr(), 0, self.loss_buf.data_ptr(), self.last_loss.data_ptr(),
                    self.losses.data_ptr(), self.losses.numel(), self.step_ctr.data_ptr(),
                    self.ticket.data_ptr(), _lib.stream_ptr()), "adam_step_tail")
                return
            m.adam_step()
            _lib.check(_lib.lib().sal_step_tail(self.loss_buf.data_ptr(),
                                                self.last_loss.data_ptr(),
                                                self.losses.data_ptr(), self.losses.numel(),
                                                self.step_ctr.data_ptr(), m.t.data_ptr(),
                                                _lib.stream_ptr()), "step_tail")

    def _pair(self, k: int, host_inputs: bool, part: str = "all") -> None:
        """{prep(slot k+1) on the prep stream || train(slot k)} on the current stream."""
        D = self.depth
        if part == "post":
            self._train(self.slots[k % D], "post")
            return

        def stg(j):  # the staging slot holding step j's inputs (end-to-end mode)
            return self.staging[j % self.ring] if host_inputs else None
        cs = torch.cuda.current_stream()
        ps = self.prep_stream or cs  # None: prep serialised on the compute stream
        split = self.cfg.late_prep and self.prep_stream is not None
        ps.wait_stream(cs)
        ls = None
        if split:
            ls = self.late_stream
            ls.wait_stream(cs)
            with torch.cuda.stream(ls):
                # the late stream also zeroes the tcgen05 gradient blocks (the previous
                # step's Adam has read them): no memset node in the training chain
                self._prep_late(self.slots[k % D], stg(k), zero_grads=True)
        with torch.cuda.stream(ps):
            self._prep(self.slots[(k + 1) % D], stg(k + 1), late=not split)
        self._train(self.slots[k % D], part, late=ls)
        cs.wait_stream(ps)

    # ---------------------------------------------------------------- driver
    def _stage_host(self, stage: _Staging, step: int) -> None:
        """End-to-end mode: one step's seeds + descriptor into pinned staging."""
        if step < len(self.desc_host):
            bid, off, n = (int(v) for v in self.desc_host[step])
        else:
            bid, off, n = -1, 0, 0
        stage.np[0], stage.np[1], stage.np[2] = bid, 0, n
        if n:
            stage.np[3:3 + n] = self.perm_host[off:off + n]

    def _push(self, stage: _Staging) -> None:
        """H2D of one staged step on the copy stream, a step before the replay that
        consumes it (which waits on `stage.copied`, long satisfied by then): no copy
        sits between two replays and no memcpy node inside the graph."""
        cps = self.copy_stream
        cps.wait_event(stage.ev)      # the last replay that read the device mirror
        with torch.cuda.stream(cps):
            stage.dev.copy_(stage.host, non_blocking=True)
            stage.copied.record(cps)

    def _stage_and_push(self, step: int) -> None:
        stage = self.staging[step % self.ring]
        stage.ev.synchronize()  # the replay that last read this staging slot
        self._stage_host(stage, step)
        self._push(stage)

    def begin_epoch(self, host_inputs: bool = False) -> None:
        """Prime the pipeline (eager): batch 0 into slot 0."""
        late = not (self.cfg.late_prep and self.prep_stream is not None)
        stages = []
        if host_inputs:  # steps 0 .. depth-1 (the first replay preps step depth-1)
            for j in range(self.depth):
                self._stage_and_push(j)
        for j in range(self.depth - 1):
            stage = None
            if host_inputs:
                stage = self.staging[j]
                torch.cuda.current_stream().wait_event(stage.copied)
            stages.append(stage)
        # with the late split, pair 0 builds slot 0's labels / reverse adjacency
        for sl in self.slots:   # a capture's warm-up may have left hops without their fill
            if sl.ws.plan.reset_in_aggregate:
                sl.ws.reset_tables()
        self._prep(self.slots[0], stages[0], late=late)

    def run_steps(self, start: int, count: int, host_inputs: bool = False,
                  loss_out: torch.Tensor | None = None) -> None:
        """Steps [start, start+count) (see _run_steps), on the dedicated training
        stream when one is configured, joined back to the caller's stream."""
        if self.compute_stream is None:
            self._run_steps(start, count, host_inputs, loss_out)
            return
        caller = torch.cuda.current_stream()
        self.compute_stream.wait_stream(caller)
        with torch.cuda.stream(self.compute_stream):
            self._run_steps(start, count, host_inputs, loss_out)
        caller.wait_stream(self.compute_stream)

    def _run_steps(self, start: int, count: int, host_inputs: bool = False,
                   loss_out: torch.Tensor | None = None) -> None:
        """Steps [start, start+count): step k trains slot k%2 and prepares k+1.

        begin_epoch() must have prepared step `start` (the pipeline is primed
        once per epoch).  With host_inputs each step stages the seeds + descriptor
        of step k+depth in pinned host memory and copies them H2D on the copy
        stream (a ring of 2*depth slots, so the host runs ahead of the GPU), and
        copies its loss back to `loss_out[k]` (pinned) — the end-to-end path.
        """
        D = self.depth
        P = self.ring if host_inputs else D
        cs = torch.cuda.current_stream()
        for k in range(start, start + count):
            if host_inputs:
                # replay k preps step k+D-1 (pushed one iteration ago); push step k+D now
                self._stage_and_push(k + D)
                cs.wait_event(self.staging[(k + D - 1) % self.ring].copied)
            if self.cfg.graphs:
                if self.graph_allreduce:
                    key = (k % P, host_inputs, "all")
                    g = self.graphs.get(key) or self._capture(k % P, host_inputs, "all")
                    if g is not None:
                        g.replay()
                        self.kernel_launches += self.graph_kernels[key]
                if not self.graph_allreduce:  # NCCL refused capture: two graphs per step
                    for part in ("pre", "post"):
                        key = (k % P, host_inputs, part)
                        g = self.graphs.get(key) or self._capture(k % P, host_inputs, part)
                        g.replay()
                        self.kernel_launches += self.graph_kernels[key]
                        if part == "pre":
                            allreduce_mean(self.model.grad, self.world)
            else:
                n0 = _lib.lib().sal_launch_count()
                self._pair(k % P, host_inputs)
                self.kernel_launches += _lib.lib().sal_launch_count() - n0
            if host_inputs:
                # step k's inputs are fully consumed (prep of k, labels of k in this replay)
                self.staging[k % self.ring].ev.record(cs)
            if loss_out is not None:
                # loss D2H on the copy stream from the step's slot of the device log, so
                # the next replay does not queue behind it
                done = self._loss_ev[k % len(self._loss_ev)]
                done.record(cs)
                self.copy_stream.wait_event(done)
                with torch.cuda.stream(self.copy_stream):
                    loss_out[k - start].copy_(self.losses[k], non_blocking=True)

    def _capture(self, parity: int, host_inputs: bool, part: str = "all"):
        """Capture one step variant without disturbing the training state.

        Returns None (and switches to the split "pre"/"post" graphs) when the
        all-reduce cannot be captured."""
        torch.cuda.synchronize()
        state = [self.cursor, self.step_ctr, self.loss_buf] + self.model.optimizer_tensors()
        # the slots too: a warm-up re-runs a tail on a half-prepared slot (depth 3)
        state += [t for sl in self.slots for t in (sl.ws.buf, sl.desc)]
        saved = [s.clone() for s in state]
        side = torch.cuda.Stream(device=self.device)
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):  # warm-up on a side stream (cuBLAS workspaces)
            for _ in range(2):
                self._pair(parity, host_inputs, part)
                if part == "pre":
                    allreduce_mean(self.model.grad, self.world)
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        n0 = _lib.lib().sal_launch_count()
        try:
            with torch.cuda.graph(g):
                self._pair(parity, host_inputs, part)
        except Exception:
            if part != "all" or self.world == 1:
                raise
            torch.cuda.synchronize()
            self.graph_allreduce = False
            for a, b in zip(state, saved):
                a.copy_(b)
            self.model.refresh_shadow()
            return None
        torch.cuda.synchronize()
        # library kernels per replay (the graph re-executes exactly these)
        self.graph_kernels[(parity, host_inputs, part)] = _lib.lib().sal_launch_count() - n0
        # undo the warm-up's side effects (cursor, counters, weights, Adam state)
        for a, b in zip(state, saved):
            a.copy_(b)
        self.model.refresh_shadow()
        self.graphs[(parity, host_inputs, part)] = g
        return g

    def train_epoch(self, epoch: int) -> float:
        n = self.set_epoch(epoch)
        self.begin_epoch()
        self.run_steps(0, n)
        torch.cuda.synchronize()
        return float(self.losses[:n].mean().item()) if n else 0.0

    # ---------------------------------------------------------------- eval
    def evaluate(self, ids: np.ndarray, fanouts: FanoutSpec | None = None,
                 batch_size: int | None = None) -> tuple[int, int]:
        """Sampled inference over `ids` on the device pipeline (Evaluator);
        returns (correct, total) summed over ranks when world > 1."""
        fan = fanouts or self.cfg.fanouts
        bs = batch_size or self.cfg.batch_size
        key = (tuple(fan.per_hop), bs)
        ev = self._evaluators.get(key) if hasattr(self, "_evaluators") else None
        if ev is None:
            self._evaluators = getattr(self, "_evaluators", {})
            ev = Evaluator(self.dg, self.model, fan, bs, self.cfg.global_seed + 7,
                           rank=self.rank, world=self.world, rng_policy=self.cfg.rng_policy,
                           graphs=self.cfg.graphs, act_dtype=self.cfg.act_dtype,
                           fuse_last_hop=self.cfg.fuse_last_hop)
            self._evaluators[key] = ev
        return ev.run(ids)

    @torch.no_grad()
    def evaluate_eager(self, ids: np.ndarray, fanouts: FanoutSpec | None = None,
                       batch_size: int | None = None) -> tuple[int, int]:
        """Sampled inference through the public prep API (run_epoch_prep ->
        materialised features -> FusedSAGE.predict), one batch at a time; the
        comparator of the Evaluator fast path (this rank's ids only)."""
        from .prep import EpochPlan, PrepConfig, run_epoch_prep
        from .sampler import SeedBatch
        fan = fanouts or self.cfg.fanouts
        bs = batch_size or self.cfg.batch_size
        ids = np.asarray(ids, dtype=np.int64)
        batches = tuple(SeedBatch(i, ids[s:s + bs]) for i, s in enumerate(range(0, len(ids), bs)))
        plan = EpochPlan(batches=batches, batch_size=bs, shuffle_seed=0)
        correct = torch.zeros((), dtype=torch.int64, device=self.device)
        total = 0
        x = _model_table(self.dg)   # the model's (padded) input width
        cfg = PrepConfig(num_workers=2, fanouts=fan, feature_dtype="bf16")
        for pb in run_epoch_prep(self.dg, x, self.dg.labels, plan, cfg, self.cfg.global_seed + 7):
            adjs = [(l.indptr, l.src_local, l.num_dst, None) for l in pb.mfg.layers]
            logits = self.model.predict(pb.features, adjs)
            correct += (logits.argmax(dim=-1) == pb.labels).sum()
            total += len(pb.labels)
        return int(correct.item()), total


class Evaluator:
    """Sampled inference over a node set on the device pipeline (
    PAPER.md:1428-1439, inference fanout (20,20,20) in the paper).

    Batches are `ids` chunked in order (batch_id = chunk index, no shuffle),
    sampled with `global_seed`; chunk b runs on rank b % world.  Three slots, each
    step one captured graph of three independent chains:
      hops(k+2):   plan cursor -> MFG hops 0..L-2      (latency-bound; hop stream)
      fill(k+1):   fused last hop -> [mean | self], labels  (HBM-bound; fill stream)
      forward(k):  SAGE layers without dropout, argmax + correct count
    so batch k+2's dependent hop kernels run under batch k+1's row traffic instead
    of before it.  The (correct, total) pair stays on the device until the end of
    the pass (one D2H; one all-reduce when world > 1).
    """

    def __init__(self, dg: DeviceGraph, model: FusedSAGE, fanouts: FanoutSpec, batch_size: int,
                 global_seed: int, rank: int = 0, world: int = 1, rng_policy: str = "splitmix",
                 graphs: bool = True, act_dtype: torch.dtype = torch.bfloat16,
                 prep_priority: int = -1, fuse_last_hop: bool = True):
        _lib.require_cuda()
        self.dg, self.model = dg, model
        self.fanouts, self.batch_size, self.global_seed = fanouts, int(batch_size), int(global_seed)
        self.rank, self.world = rank, world
        self.device = dg.device
        self.nh = len(fanouts)
        self.policy = RNG_POLICIES[rng_policy]
        self.use_graphs = graphs
        cfg = TrainConfig(fanouts=fanouts, batch_size=self.batch_size, gather_free=True,
                          act_dtype=act_dtype, fuse_last_hop=fuse_last_hop)
        self.D = 3
        self.slots = [_Slot(dg, cfg, self.device, backward=False) for _ in range(self.D)]
        # the hop chain at high priority (latency-bound: its blocks go first as the row
        # traffic's blocks drain); the fill at the default
        self.hop_stream = torch.cuda.Stream(device=self.device, priority=prep_priority)
        self.fill_stream = torch.cuda.Stream(device=self.device)
        self.x_table = _model_table(dg)
        self.cursor = torch.zeros(1, dtype=torch.int64, device=self.device)
        self.counts = torch.zeros(2, dtype=torch.int64, device=self.device)
        self.seeds_all = torch.zeros(1, dtype=torch.int64, device=self.device)
        self.desc_all = torch.zeros((1, 3), dtype=torch.int64, device=self.device)
        self.n_steps = 0
        self.graphs = {}
        self.graph_kernels = {}
        self.kernel_launches = 0

    def set_ids(self, ids: np.ndarray, check: bool = True) -> int:
        """Chunk and shard `ids`, upload seeds + descriptors; returns this rank's steps.
        check=False leaves the distinct-seeds check to the caller (run() does it on the
        host while the pass runs)."""
        ids = np.ascontiguousarray(np.asarray(ids, dtype=np.int64).reshape(-1))
        self._ids = ids
        bs = self.batch_size
        descs = chunk_descs(ids, bs, self.rank, self.world, check=check)
        n = len(descs)
        if self.seeds_all.numel() < max(1, len(ids)):
            self.seeds_all = torch.zeros(len(ids), dtype=torch.int64, device=self.device)
            self.graphs.clear()
        if self.desc_all.shape[0] < max(1, n) or self.n_steps != n:
            self.desc_all = torch.zeros((max(1, n), 3), dtype=torch.int64, device=self.device)
            self.graphs.clear()
        if len(ids):
            self.seeds_all[:len(ids)].copy_(torch.from_numpy(ids))
        if n:
            self.desc_all[:n].copy_(torch.from_numpy(np.asarray(descs, np.int64)))
        self.n_steps = n
        return n

    def _hops(self, slot: _Slot) -> None:
        """Plan cursor -> the slot's descriptor -> MFG hops (the fused last hop is left
        to _fill)."""
        st = torch.cuda.current_stream()
        # a separate cursor kernel here: with the 3-slot pipeline the folded form
        # (sal_sample_mfg_next, one seed-insertion block) measured 0.0534 vs 0.0527 s
        L = _lib.lib()
        _lib.check(L.sal_plan_next(self.desc_all.data_ptr(), self.n_steps, self.cursor.data_ptr(),
                                   slot.desc.data_ptr(), _lib.stream_ptr(st)), "plan_next")
        slot.ws.run(self.dg, self.seeds_all, slot.desc, self.global_seed, self.policy, st)

    def _fill(self, slot: _Slot) -> None:
        """The layer-0 input (fused last hop, or the destination rows) and the labels."""
        ws = slot.ws
        st = torch.cuda.current_stream()
        L = _lib.lib()
        nh = self.nh
        f, fx = self.model.dims[0], self.x_table.shape[1]
        if slot.fused:
            ws.aggregate(self.dg, self.x_table, slot.feats, f, slot.desc, self.global_seed,
                         self.policy, st)
        else:
            gather_rows(self.x_table, ws.globals, slot.feats[:, f:f + fx],
                        n=ws.node_cap[nh - 1], n_dev=ws.sizes[nh - 1:nh], stream=st)
        _lib.check(L.sal_gather_labels(self.dg.labels.data_ptr(), self.seeds_all.data_ptr(),
                                       slot.desc.data_ptr(), self.batch_size,
                                       slot.labels.data_ptr(), _lib.stream_ptr(st)),
                   "gather_labels")

    def _forward(self, slot: _Slot) -> None:
        ws = slot.ws
        adjs = []
        for i in range(self.nh):
            h = self.nh - 1 - i
            adjs.append((ws.dst_indptr[h], ws.src_local[h], ws.node_cap[h], ws.sizes[h:h + 1]))
        m = self.model
        was = m.training
        m.training = False
        head = m.head_ok()
        try:
            xg = None if slot.fused else (self.x_table, ws.src_glob)
            logits, saved = m.forward(slot.feats, adjs, x_global=xg, head=head,
                                      mean0_ready=slot.fused)
        finally:
            m.training = was
        if head:   # logits stay in TMEM: argmax + correct count in the GEMM's epilogue
            m.score(saved, slot.labels, self.counts)
            return
        _lib.check(_lib.lib().sal_argmax_correct(
            logits.data_ptr(), logits.stride(0), min(logits.shape[0], self.batch_size),
            logits.shape[1], _lib.dtype_code(logits.dtype), slot.labels.data_ptr(),
            self.counts.data_ptr(), None, _lib.stream_ptr()), "argmax_correct")

    def _pair(self, k: int) -> None:
        """{hops(k+2) || fill(k+1) || forward(k)} (begin() primed hops/fill of k, hops
        of k+1)."""
        D = self.D
        cs = torch.cuda.current_stream()
        hs, fs = self.hop_stream, self.fill_stream
        hs.wait_stream(cs)
        fs.wait_stream(cs)
        with torch.cuda.stream(hs):
            self._hops(self.slots[(k + 2) % D])
        with torch.cuda.stream(fs):
            self._fill(self.slots[(k + 1) % D])
        self._forward(self.slots[k % D])
        cs.wait_stream(hs)
        cs.wait_stream(fs)

    def _prime(self) -> None:
        """Step 0's hops and fill, step 1's hops (eager, current stream).  A slot's hops
        rely on the fill of its previous batch to have reset its id table; a capture's
        warm-up leaves hops without their fill, so every table is reset here."""
        for s in self.slots:
            if s.ws.plan.reset_in_aggregate:
                s.ws.reset_tables()
        self._hops(self.slots[0])
        self._fill(self.slots[0])
        self._hops(self.slots[1 % self.D])

    def _capture(self, parity: int):
        torch.cuda.synchronize()
        saved = (self.cursor.clone(), self.counts.clone())
        side = torch.cuda.Stream(device=self.device)
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            # warm-up along a valid pipeline progression: each pair reads slots the
            # previous ones prepared
            self._prime()
            for k in range(parity + 1):
                self._pair(k)
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        n0 = _lib.lib().sal_launch_count()
        with torch.cuda.graph(g):
            self._pair(parity)
        torch.cuda.synchronize()
        self.graph_kernels[parity] = _lib.lib().sal_launch_count() - n0
        self.cursor.copy_(saved[0])
        self.counts.copy_(saved[1])
        self.graphs[parity] = g
        return g

    def capture_all(self) -> None:
        """Capture every slot parity's graph (before begin(): capturing replays steps)."""
        if self.use_graphs:
            for p in range(min(self.D, max(self.n_steps, 1))):
                if p not in self.graphs:
                    self._capture(p)

    def begin(self) -> None:
        """Reset the cursor and counters and prime the pipeline for step 0."""
        self.cursor.zero_()
        self.counts.zero_()
        self._prime()

    def steps(self, start: int, count: int) -> None:
        """Enqueue steps [start, start+count) (begin() primed step `start`)."""
        D = self.D
        for k in range(start, start + count):
            if self.use_graphs:
                g = self.graphs.get(k % D) or self._capture(k % D)
                g.replay()
                self.kernel_launches += self.graph_kernels[k % D]
            else:
                n0 = _lib.lib().sal_launch_count()
                self._pair(k)
                self.kernel_launches += _lib.lib().sal_launch_count() - n0

    def run(self, ids: np.ndarray) -> tuple[int, int]:
        n = self.set_ids(ids, check=False)
        self.capture_all()   # before the pass: capturing replays steps
        self.begin()
        self.steps(0, n)
        # the seeds' distinct check runs on the host under the device pass; a failure
        # raises before any result is read (every rank checks every chunk alike)
        check_chunks_distinct(self._ids, self.batch_size)
        if self.world > 1:
            torch.distributed.all_reduce(self.counts)
        c, t = self.counts.tolist()
        return int(c), int(t)
