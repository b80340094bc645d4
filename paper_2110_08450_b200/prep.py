"""On-device batch preparation (drop-in for mfgprep.prep, prep.py:1-357).

The reference prepares batches with P CPU threads, a bounded queue and a
pool of reusable host buffers (prep.py:226-334).  Here every batch is
prepared by GPU-wide kernels; `num_workers` batches are prepared concurrently
on their own CUDA streams and `depth` batches are in flight ahead of the
consumer, each in its own device slot (MFG workspace
+ feature + label buffers), so sampling/slicing of batch i+1.. overlaps
whatever the consumer runs for batch i on its own stream.  A slot is
recycled only after the consumer stream has passed an event recorded when
the consumer advanced (the same "borrowed until the iterator advances"
contract as prep.py:11-13).

Names, arguments and errors mirror the reference: `make_epoch_plan`,
`EpochPlan`, `PrepConfig`, `PreparedBatch`, `slice_features`,
`slice_labels`, `prepare_batch`, `PrepReport`, `EpochPrepRun`,
`run_epoch_prep`, `prep_sweep_csv`.
"""

from __future__ import annotations

import hashlib
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .graph import (DeviceGraph, FeatureMatrix, LabelVector, as_device_graph, upload_features,
                    upload_labels)
from .sampler import (FanoutSpec, IdMap, Mfg, MfgWorkspace, RNG_POLICIES, SamplerVariant,
                      SeedBatch)


@dataclass(frozen=True)
class EpochPlan:
    batches: tuple
    batch_size: int
    shuffle_seed: int

    def __len__(self):
        return len(self.batches)


def make_epoch_plan(train_ids, batch_size: int, shuffle_seed: int) -> EpochPlan:
    """PCG64 shuffle of train ids, chunked into SeedBatches (prep.py:40-52).

    Same numpy call as the reference, so batch ids and seeds are identical.
    """
    if batch_size < 1:
        raise ValueError("batch_size must be >= 1")
    ids = np.asarray(train_ids, dtype=np.int64).reshape(-1)
    perm = ids[np.random.default_rng(shuffle_seed).permutation(len(ids))]
    starts = range(0, len(perm), batch_size)
    return EpochPlan(batches=tuple(SeedBatch(i, perm[s:s + batch_size])
                                   for i, s in enumerate(starts)),
                     batch_size=batch_size, shuffle_seed=shuffle_seed)


@dataclass
class PrepConfig:
    """prep.py:55-72.  On the GPU `num_workers` is the number of batches
    prepared concurrently (one CUDA stream each) and ahead of the consumer."""

    num_workers: int = 1
    queue_capacity: int = 0
    fanouts: FanoutSpec = field(default_factory=lambda: FanoutSpec((15, 10, 5)))
    variant: SamplerVariant = field(default_factory=SamplerVariant)
    delivery: str = "in_order"
    feature_dtype: str = "f32"      # output dtype of the sliced features
    rng_policy: str = "splitmix"
    # each batch as two CUDA-graph replays (sample | slice) instead of ~15 host launches;
    # the slots, streams and graphs of a run are kept for the next run of the same shape
    graphs: bool = True

    def __post_init__(self):
        if self.num_workers < 1:
            raise ValueError("need at least one worker")
        if self.queue_capacity == 0:
            self.queue_capacity = 4 * self.num_workers
        if self.queue_capacity < 1:
            raise ValueError("queue capacity must be >= 1")
        if self.delivery not in ("in_order", "completion_order"):
            raise ValueError(f"unknown delivery mode {self.delivery!r}")
        if self.feature_dtype not in ("f32", "f16", "bf16"):
            raise ValueError(f"unknown feature dtype {self.feature_dtype!r}")
        if self.rng_policy not in RNG_POLICIES:
            raise ValueError(f"unknown rng policy {self.rng_policy!r}")

    @property
    def depth(self) -> int:
        """Batches in flight ahead of the consumer: up to two per worker stream (so a
        worker's next batch is already queued on its stream when the current one ends,
        like a reference worker that moves on while the consumer holds its batch),
        within the reference's pool of queue_capacity + num_workers buffers
        (prep.py:239; the consumer's current batch holds one)."""
        return max(1, min(2 * self.num_workers, self.num_workers + self.queue_capacity - 1))


_TORCH_DT = {"f32": torch.float32, "f16": torch.float16, "bf16": torch.bfloat16}


@dataclass
class PreparedBatch:
    """An Mfg joined with sliced features/labels, resident in HBM (prep.py:112-150)."""

    mfg: Mfg
    features: torch.Tensor   # (num_nodes, f) on device
    labels: torch.Tensor     # (|seeds|,) int64 on device
    byte_size: int
    stats: tuple
    _slot: object = None
    _run: object = None

    @property
    def num_nodes(self) -> int:
        return self.mfg.num_nodes

    @property
    def num_edges(self) -> int:
        return self.mfg.num_edges

    def digest(self) -> str:
        """prep.py:132-137 over host copies (features as f32, labels int64)."""
        h = hashlib.blake2b(digest_size=16)
        h.update(self.mfg.digest().encode())
        h.update(np.ascontiguousarray(self.features.float().cpu().numpy()).tobytes())
        h.update(np.ascontiguousarray(self.labels.cpu().numpy().astype(np.int64)).tobytes())
        return h.hexdigest()

    def detach(self) -> "PreparedBatch":
        """Copy out of the slot and release it (prep.py:139-145)."""
        idm = _detached_idmap(self.mfg.id_map)
        layers = tuple(type(l)(l.num_dst, l.num_src, l.indptr.clone(), l.src_local.clone())
                       for l in self.mfg.layers)
        out = PreparedBatch(mfg=Mfg(layers=layers, id_map=idm, seeds=self.mfg.seeds),
                            features=self.features.clone(), labels=self.labels.clone(),
                            byte_size=self.byte_size, stats=self.stats)
        self.release()
        return out

    def release(self):
        if self._run is not None and self._slot is not None:
            self._run._release(self._slot)
        self._slot = None
        self._run = None


def _detached_idmap(m: IdMap) -> IdMap:
    g = m.global_ids.clone()
    t = m._table.clone()
    return IdMap(m.variant, device=g.device, _table=t, _globals=g, _size=m.size)


def _feature_source(fm):
    """Device [n, f] feature view for a FeatureMatrix / DeviceGraph / tensor."""
    if isinstance(fm, DeviceGraph):
        return fm.feature_view()
    if isinstance(fm, torch.Tensor):
        return fm
    return upload_features(fm)


def _label_source(y):
    if isinstance(y, DeviceGraph):
        return y.labels
    if isinstance(y, torch.Tensor):
        return y
    return upload_labels(y)


def gather_rows(x: torch.Tensor, ids: torch.Tensor, out: torch.Tensor, n: int | None = None,
                n_dev: torch.Tensor | None = None, stream=None) -> None:
    """out[i,:] = x[ids[i],:] through sal_gather_rows (row count n or *n_dev)."""
    L = _lib.lib()
    if ids.dtype not in (torch.int32, torch.int64):
        raise ValueError("ids must be int32 or int64")
    rows = n if n is not None else out.shape[0]
    _lib.check(L.sal_gather_rows(x.data_ptr(), x.shape[0], x.shape[1], x.stride(0),
                                 _lib.dtype_code(x.dtype), ids.data_ptr(), ids.element_size(),
                                 _lib.ptr(n_dev), rows, out.data_ptr(), out.stride(0),
                                 _lib.dtype_code(out.dtype), _lib.stream_ptr(stream)),
               "gather_rows")


def slice_features(fm, id_map: IdMap, out: torch.Tensor) -> torch.Tensor:
    """Gather id_map's rows into `out` as f32 (prep.py:153-171).

    `out` must be a float32 device buffer holding >= size * cols elements;
    raises ValueError on a shortfall rather than truncating.
    """
    x = _feature_source(fm)
    cols = x.shape[1]
    need = id_map.size * cols
    if out.dtype != torch.float32:
        raise ValueError("output buffer must be float32")
    if out.numel() < need:
        raise ValueError(f"output buffer holds {out.numel()} elements, need {need}")
    view = out.reshape(-1)[:need].view(id_map.size, cols)
    if need:
        gather_rows(x, id_map._globals, view, n=id_map.size)
    return view


def slice_labels(y, seeds: SeedBatch, out: torch.Tensor | None = None) -> torch.Tensor:
    """Destination labels in seed order (prep.py:174-182)."""
    vals = _label_source(y)
    n = len(seeds)
    if out is None:
        out = torch.empty(n, dtype=torch.int64, device=vals.device)
    view = out[:n]
    if n:
        idx = torch.from_numpy(seeds.dst_ids).to(vals.device)
        torch.index_select(vals, 0, idx, out=view)
    return view


def _batch_bytes(mfg: Mfg, cols: int, nseeds: int) -> int:
    """prep.py:185-189 accounting (features as f32, labels/edges as int64)."""
    edges = sum(8 * l.num_edges + 8 * (l.num_dst + 1) for l in mfg.layers)
    return mfg.num_nodes * cols * 4 + nseeds * 8 + edges


class _Slot:
    """Device buffers for one in-flight batch (the BufferPool slot, prep.py:75-109)."""

    def __init__(self, dg: DeviceGraph, cfg: PrepConfig, max_seeds: int, cols: int, device):
        self.ws = MfgWorkspace(dg.num_nodes, cfg.fanouts, max_seeds, device=device)
        n_cap = self.ws.node_cap[-1]
        self.features = torch.empty((max(n_cap, 1), max(cols, 1)),
                                    dtype=_TORCH_DT[cfg.feature_dtype], device=device)
        self.labels = torch.empty(max(max_seeds, 1), dtype=torch.int64, device=device)
        self.extents = torch.empty(2 * cfg.fanouts.__len__() + 1, dtype=torch.int64,
                                   pin_memory=True)
        self.ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        self.done = torch.cuda.Event()
        self.free = torch.cuda.Event()
        self.seeds = None
        self.index = -1


def _prep_into_slot(dg, x, yv, slot: _Slot, seeds: SeedBatch, seeds_base: torch.Tensor,
                    desc: torch.Tensor, global_seed: int, policy: int, stream) -> None:
    """Enqueue sample + slice for one batch into `slot` on `stream`.

    seeds_base/desc are device-resident (sal_batch_desc), so nothing here
    blocks the host: the whole batch is asynchronous work on `stream`.
    """
    ws = slot.ws
    with torch.cuda.stream(stream):
        stream.wait_event(slot.free)
        slot.ev[0].record(stream)
        ws.run(dg, seeds_base, desc, global_seed, policy, stream)
        slot.ev[1].record(stream)
        n_nodes = ws.sizes[ws.num_hops:ws.num_hops + 1]
        if x is not None:
            gather_rows(x, ws.globals, slot.features[:, :x.shape[1]], n=ws.node_cap[-1],
                        n_dev=n_nodes, stream=stream)
        if yv is not None and len(seeds):
            L = _lib.lib()
            _lib.check(L.sal_gather_labels(yv.data_ptr(), seeds_base.data_ptr(), desc.data_ptr(),
                                           len(seeds), slot.labels.data_ptr(),
                                           _lib.stream_ptr(stream)), "gather_labels")
        slot.ev[2].record(stream)
        slot.extents.copy_(torch.cat([ws.sizes, ws.etot]), non_blocking=True)
        slot.done.record(stream)
    slot.seeds = seeds


def _mfg_from_ws(ws: MfgWorkspace, sizes, etot, seeds: SeedBatch, variant: SamplerVariant) -> Mfg:
    """The Mfg view of a sampled workspace, given its host-known extents."""
    from .sampler import MfgLayer
    nh = ws.num_hops
    layers = []
    for h in range(nh):
        nd = sizes[h]
        layers.append(MfgLayer(num_dst=nd, num_src=sizes[h + 1],
                               indptr=ws.dst_indptr[h][:nd + 1],
                               src_local=ws.src_local[h][:etot[h]]))
    idm = IdMap(variant, device=ws.device, _table=ws.table, _globals=ws.globals,
                _size=sizes[-1])
    return Mfg(layers=tuple(reversed(layers)), id_map=idm, seeds=seeds, workspace=ws)


def _finish_slot(slot: _Slot, cols: int, variant: SamplerVariant, run=None) -> PreparedBatch:
    slot.done.synchronize()
    ws = slot.ws
    ext = slot.extents.tolist()
    nh = ws.num_hops
    sizes, etot = ext[:nh + 1], ext[nh + 1:]
    mfg = _mfg_from_ws(ws, sizes, etot, slot.seeds, variant)
    feats = slot.features[:sizes[-1], :cols]
    labels = slot.labels[:len(slot.seeds)]
    stats = tuple((l.num_dst, l.num_src, l.num_edges) for l in mfg.layers)
    return PreparedBatch(mfg=mfg, features=feats, labels=labels,
                         byte_size=_batch_bytes(mfg, cols, len(slot.seeds)), stats=stats,
                         _slot=slot if run is not None else None, _run=run)


def prepare_batch(g, fm, y, seeds: SeedBatch, fanouts: FanoutSpec, variant: SamplerVariant,
                  global_seed: int, slot=None, pool=None, *, feature_dtype: str = "f32",
                  rng_policy: str = "splitmix") -> PreparedBatch:
    """Sample the MFG then slice features and labels for one batch (prep.py:192-206).

    Like the reference, the MFG is built first and the feature/label buffers are then
    sized to it (its _Slot.reserve): one MFG workspace plus exactly num_nodes x cols
    feature rows, not a worst-case node_cap buffer.  A `slot` from this module (the
    buffers of an epoch run, or one the caller keeps) is reused instead; `pool` is
    accepted for signature compatibility (slots are recycled by run_epoch_prep)."""
    dg = as_device_graph(g)
    x = _feature_source(fm) if fm is not None else None
    yv = _label_source(y) if y is not None else None
    cols = x.shape[1] if x is not None else 0
    stream = torch.cuda.current_stream()
    policy = RNG_POLICIES[rng_policy]
    if isinstance(slot, _Slot):
        if slot.ws.fanouts != fanouts or slot.ws.max_seeds < len(seeds):
            raise ValueError("slot was built for other fanouts or a smaller batch")
        slot.ws.load_seeds(seeds, stream)
        _prep_into_slot(dg, x, yv, slot, seeds, slot.ws.seeds, slot.ws.desc, global_seed,
                        policy, stream)
        return _finish_slot(slot, cols, variant)
    ws = MfgWorkspace(dg.num_nodes, fanouts, len(seeds), device=dg.device)
    ws.load_seeds(seeds, stream)
    ws.run(dg, ws.seeds, ws.desc, global_seed, policy, stream)
    sizes, etot = ws.read_extents()
    n = sizes[-1]
    feats = torch.empty((n, cols), dtype=_TORCH_DT[feature_dtype], device=dg.device)
    if x is not None and n:
        gather_rows(x, ws.globals, feats, n=n, stream=stream)
    labels = torch.empty(len(seeds), dtype=torch.int64, device=dg.device)
    if yv is not None and len(seeds):
        _lib.check(_lib.lib().sal_gather_labels(yv.data_ptr(), ws.seeds.data_ptr(),
                                                ws.desc.data_ptr(), len(seeds),
                                                labels.data_ptr(), _lib.stream_ptr(stream)),
                   "gather_labels")
    mfg = _mfg_from_ws(ws, sizes, etot, seeds, variant)
    stats = tuple((l.num_dst, l.num_src, l.num_edges) for l in mfg.layers)
    return PreparedBatch(mfg=mfg, features=feats, labels=labels,
                         byte_size=_batch_bytes(mfg, cols, len(seeds)), stats=stats)


@dataclass
class PrepReport:
    """prep.py:209-223; durations from CUDA events on the prep stream."""

    threads: int
    sampling_s: float = 0.0
    slicing_s: float = 0.0
    both_s: float = 0.0
    per_batch: list = field(default_factory=list)
    peak_resident: int = 0

    def csv_row(self) -> str:
        return f"{self.threads},{self.sampling_s:.6f},{self.slicing_s:.6f},{self.both_s:.6f}"

    @staticmethod
    def csv_header() -> str:
        return "threads,sampling_s,slicing_s,both_s"


class _EpochResources:
    """Slots, streams, plan buffers and per-slot CUDA graphs of one run shape, kept
    across runs of the same (graph, features, labels, config, seed): a second epoch
    allocates nothing and captures nothing."""

    def __init__(self, dg, x, yv, cfg: PrepConfig, max_seeds: int, cols: int, n_ids: int,
                 nb: int, global_seed: int):
        dev = dg.device
        self.depth = cfg.depth
        self.slots = [_Slot(dg, cfg, max_seeds, cols, dev) for _ in range(self.depth + 1)]
        self.streams = [torch.cuda.Stream(device=dev)
                        for _ in range(max(1, min(cfg.num_workers, self.depth)))]
        # plan buffers with headroom (the graphs hold their addresses): any epoch of up
        # to 2048 batches reuses them
        nb_cap = max(nb, 2048)
        ids_cap = max(n_ids, min(nb_cap * max_seeds, 1 << 24))
        self.seeds_all = torch.zeros(max(ids_cap, 1), dtype=torch.int64, device=dev)
        self.desc_all = torch.zeros((nb_cap, 3), dtype=torch.int64, device=dev)
        self.max_seeds = max_seeds
        self.graphed = False

    def fits(self, max_seeds: int, n_ids: int, nb: int) -> bool:
        return (max_seeds <= self.max_seeds and n_ids <= self.seeds_all.numel()
                and nb <= self.desc_all.shape[0])

    def capture(self, dg, x, yv, global_seed: int, policy: int) -> None:
        """Per slot: g_sample = {plan cursor -> slot desc, MFG build}, g_slice = {row
        gather, labels, extents D2H}.  The cursor (one int64) is the only per-batch input."""
        n_cap = self.desc_all.shape[0]
        L = _lib.lib()
        torch.cuda.synchronize()
        for slot in self.slots:
            ws = slot.ws
            slot.cursor = torch.zeros(1, dtype=torch.int64, device=ws.device)
            slot.cursor_host = torch.zeros(1, dtype=torch.int64, pin_memory=True)
            slot.gdesc = torch.zeros(3, dtype=torch.int64, device=ws.device)
            nh = ws.num_hops
            gs, gl = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
            with torch.cuda.graph(gs):
                _lib.check(L.sal_plan_next(self.desc_all.data_ptr(), n_cap,
                                           slot.cursor.data_ptr(), slot.gdesc.data_ptr(),
                                           _lib.stream_ptr()), "plan_next")
                ws.run(dg, self.seeds_all, slot.gdesc, global_seed, policy)
            with torch.cuda.graph(gl):
                if x is not None:
                    gather_rows(x, ws.globals, slot.features[:, :x.shape[1]], n=ws.node_cap[-1],
                                n_dev=ws.sizes[nh:nh + 1])
                if yv is not None and self.max_seeds:
                    _lib.check(L.sal_gather_labels(yv.data_ptr(), self.seeds_all.data_ptr(),
                                                   slot.gdesc.data_ptr(), self.max_seeds,
                                                   slot.labels.data_ptr(), _lib.stream_ptr()),
                               "gather_labels")
                slot.extents[:nh + 1].copy_(ws.sizes, non_blocking=True)
                slot.extents[nh + 1:].copy_(ws.etot, non_blocking=True)
            slot.g_sample, slot.g_slice = gs, gl
        torch.cuda.synchronize()
        self.graphed = True


_RES_CACHE: dict = {}


def release_prep_cache() -> None:
    """Free the slots and graphs run_epoch_prep keeps for the next run."""
    _RES_CACHE.clear()


def _resources(dg, x, yv, cfg: PrepConfig, max_seeds: int, cols: int, n_ids: int, nb: int,
               global_seed: int) -> _EpochResources:
    key = (id(dg), None if x is None else (x.data_ptr(), tuple(x.shape), x.stride(0), x.dtype),
           None if yv is None else yv.data_ptr(), tuple(cfg.fanouts.per_hop), cfg.feature_dtype,
           cfg.rng_policy, cfg.depth, cfg.num_workers, global_seed)
    res = _RES_CACHE.get(key)
    if res is None or not res.fits(max_seeds, n_ids, nb):
        _RES_CACHE.clear()   # one shape at a time: slots hold worst-case buffers
        res = _EpochResources(dg, x, yv, cfg, max_seeds, cols, n_ids, nb, global_seed)
        res.refs = (dg, x, yv)   # keep the captured pointers alive
        _RES_CACHE[key] = res
    return res


class EpochPrepRun:
    """Iterable over an epoch's PreparedBatches (prep.py:226-334)."""

    def __init__(self, g, fm, y, plan: EpochPlan, cfg: PrepConfig, global_seed: int):
        self._g, self._fm, self._y = g, fm, y
        self._plan, self._cfg, self._seed = plan, cfg, global_seed
        self.report = PrepReport(threads=cfg.num_workers)
        self._free = []
        self._resident = 0

    def _release(self, slot: _Slot):
        slot.free.record(torch.cuda.current_stream())
        self._free.append(slot)
        self._resident -= 1

    def __iter__(self):
        plan, cfg = self._plan, self._cfg
        dg = as_device_graph(self._g)
        x = _feature_source(self._fm) if self._fm is not None else None
        yv = _label_source(self._y) if self._y is not None else None
        cols = x.shape[1] if x is not None else 0
        nb = len(plan)
        t0 = time.perf_counter()
        if nb == 0:
            self.report.both_s = time.perf_counter() - t0
            return
        max_seeds = max(len(b) for b in plan.batches)
        depth = cfg.depth
        policy = RNG_POLICIES[cfg.rng_policy]
        # the whole plan goes to HBM once: seeds + one sal_batch_desc per batch
        lens = np.array([len(b) for b in plan.batches], dtype=np.int64)
        offs = np.zeros(nb, dtype=np.int64)
        offs[1:] = np.cumsum(lens)[:-1]
        descs = np.stack([np.array([b.batch_id for b in plan.batches], dtype=np.int64), offs,
                          lens], axis=1)
        n_ids = int(lens.sum())
        if cfg.graphs:
            res = _resources(dg, x, yv, cfg, max_seeds, cols, n_ids, nb, self._seed)
            slots, streams = res.slots, res.streams
            seeds_all, desc_all = res.seeds_all, res.desc_all
        else:
            res = None
            slots = [_Slot(dg, cfg, max_seeds, cols, dg.device) for _ in range(depth + 1)]
            # num_workers batches are prepared concurrently, one CUDA stream each (the
            # reference's P worker threads, prep.py:255-287)
            streams = [torch.cuda.Stream(device=dg.device)
                       for _ in range(max(1, min(cfg.num_workers, depth)))]
            seeds_all = torch.zeros(max(n_ids, 1), dtype=torch.int64, device=dg.device)
            desc_all = torch.zeros((nb, 3), dtype=torch.int64, device=dg.device)
        if n_ids:
            seeds_all[:n_ids].copy_(torch.from_numpy(np.concatenate([b.dst_ids
                                                                     for b in plan.batches])))
        desc_all[:nb].copy_(torch.from_numpy(np.ascontiguousarray(descs)))
        if res is not None and not res.graphed:
            res.capture(dg, x, yv, self._seed, policy)
        for st in streams:   # plan uploads (current stream) before any replay reads them
            st.wait_stream(torch.cuda.current_stream())
        self._free = list(slots)
        pending = []
        nxt = 0

        def launch():
            nonlocal nxt
            slot = self._free.pop()
            slot.index = nxt
            try:
                _prep_one(dg, x, yv, slot, plan.batches[nxt], seeds_all, desc_all[nxt],
                          self._seed, policy, streams[nxt % len(streams)],
                          cursor=nxt if res is not None else None)
            except Exception as exc:
                raise RuntimeError("batch preparation worker failed") from exc
            pending.append(slot)
            nxt += 1
            self._resident += 1
            self.report.peak_resident = max(self.report.peak_resident, self._resident)

        current = None
        try:
            while nxt < nb and len(pending) < depth:
                launch()
            in_order = cfg.delivery == "in_order"
            while pending:
                # in_order: plan order (prep.py:289-297); completion_order: the first
                # in-flight batch whose stream has finished it, else the oldest
                j = 0
                if not in_order:
                    j = next((i for i, sl in enumerate(pending) if sl.done.query()), 0)
                slot = pending.pop(j)
                batch = _finish_slot(slot, cols, cfg.variant, run=self)
                ts = slot.ev[0].elapsed_time(slot.ev[1]) / 1e3
                tsl = slot.ev[1].elapsed_time(slot.ev[2]) / 1e3
                self.report.per_batch.append((slot.seeds.batch_id, ts, tsl))
                self.report.sampling_s += ts
                self.report.slicing_s += tsl
                if current is not None:
                    current.release()
                current = batch
                while nxt < nb and len(pending) < depth and self._free:
                    launch()
                yield batch
        finally:
            if current is not None:
                current.release()
            for st in streams:
                torch.cuda.current_stream().wait_stream(st)
                st.synchronize()
            self.report.both_s = time.perf_counter() - t0


def _prep_one(dg, x, yv, slot, seeds, seeds_base, desc, global_seed, policy, stream,
              cursor=None):
    """Per-batch work item (module-level so tests can inject failures): the slot's two
    graph replays behind a one-word cursor upload, or (cursor None) the direct launches."""
    if cursor is None:
        _prep_into_slot(dg, x, yv, slot, seeds, seeds_base, desc, global_seed, policy, stream)
        return
    with torch.cuda.stream(stream):
        stream.wait_event(slot.free)
        slot.cursor_host[0] = cursor
        slot.cursor.copy_(slot.cursor_host, non_blocking=True)
        slot.ev[0].record(stream)
        slot.g_sample.replay()
        slot.ev[1].record(stream)
        slot.g_slice.replay()
        slot.ev[2].record(stream)
        slot.done.record(stream)
    slot.seeds = seeds


def run_epoch_prep(g, fm, y, plan: EpochPlan, cfg: PrepConfig, global_seed: int) -> EpochPrepRun:
    return EpochPrepRun(g, fm, y, plan, cfg, global_seed)


def prep_sweep_csv(g, fm, y, plan, workers_list, fanouts, variant, global_seed: int) -> str:
    """One epoch per prefetch depth; CSV of per-stage totals (prep.py:344-357)."""
    lines = [PrepReport.csv_header()]
    if len(plan):
        prepare_batch(g, fm, y, plan.batches[0], fanouts, variant, global_seed)
    for p in workers_list:
        run = run_epoch_prep(g, fm, y, plan, PrepConfig(num_workers=p, fanouts=fanouts,
                                                        variant=variant), global_seed)
        for _ in run:
            pass
        lines.append(run.report.csv_row())
    return "\n".join(lines) + "\n"
