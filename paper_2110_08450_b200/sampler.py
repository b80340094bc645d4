"""Fanout sampling and MFG construction on the GPU (drop-in for mfgprep.sampler).

Public surface mirrors /root/reference/pkg/src/mfgprep/sampler.py:
`SamplerVariant`, `list_variants`, `FanoutSpec`, `SeedBatch`, `IdMap`,
`MfgLayer`, `Mfg`, `HopStream`, `CounterRng`, `sample_neighbors`,
`one_hop_mfg`, `multihop_mfg`, `size_hint_for` — same names, argument
meaning and error behaviour.  The arrays inside the returned objects live in
HBM (torch CUDA tensors, int32); `Mfg.digest()` / `to_host()` give the
reference's int64 host view.

Every call runs hand-written sm_100a kernels through the C-ABI (_lib); there
is no CPU fallback.  The 18 `SamplerVariant`s are output-identical by the
reference's contract (SPEC.md "Cross-variant equality"), so the device path
accepts every descriptor and runs its one data-parallel implementation.
"""

from __future__ import annotations

import ctypes
import hashlib
from dataclasses import dataclass
from itertools import product

import numpy as np
import torch

from . import _lib
from .graph import DeviceGraph, as_device_graph

MASK64 = (1 << 64) - 1
_G = 0x9E3779B97F4A7C15
_M1 = 0xBF58476D1CE4E5B9
_M2 = 0x94D049BB133111EB

MAP_IMPLS = ("std_hash", "flat_probing", "flat_probing_with_size_hint")
SET_IMPLS = ("hash_set", "vector_set", "bit_set")
RNG_POLICIES = {"splitmix": _lib.SAL_RNG_SPLITMIX, "philox": _lib.SAL_RNG_PHILOX}


# ---------------------------------------------------------------------------
# keyed splitmix64 streams (reference rng.py:16-51; device copy in common.cuh)
# ---------------------------------------------------------------------------
def _fmix(z: int) -> int:
    z &= MASK64
    z = ((z ^ (z >> 30)) * _M1) & MASK64
    z = ((z ^ (z >> 27)) * _M2) & MASK64
    return z ^ (z >> 31)


def _fmix_inverse(z: int) -> int:
    """Inverse of the splitmix64 finalizer (a bijection on 64-bit words)."""
    z &= MASK64
    z ^= z >> 31 ^ z >> 62
    z = (z * pow(_M2, -1, 1 << 64)) & MASK64
    z ^= z >> 27 ^ z >> 54
    z = (z * pow(_M1, -1, 1 << 64)) & MASK64
    z ^= z >> 30 ^ z >> 60
    return z


def hop_key_prefix(global_seed: int, batch_id: int, hop: int) -> int:
    return _fmix(_fmix(_fmix(global_seed ^ _G) ^ batch_id) ^ (hop + 0x51ED))


def stream_key(global_seed: int, batch_id: int, hop: int, dst_pos: int) -> int:
    return _fmix(hop_key_prefix(global_seed, batch_id, hop) ^ dst_pos)


class CounterRng:
    """Draw-counter view over one keyed stream (rng.py:38-51)."""

    def __init__(self, key: int):
        self.key = key & MASK64
        self.counter = 0

    def next_u64(self) -> int:
        self.counter += 1
        return _fmix(self.key + self.counter * _G)

    def next_below(self, n: int) -> int:
        return self.next_u64() % n


class HopStream:
    """Key context for one (global_seed, batch_id, hop) pass (sampler.py:238-250)."""

    def __init__(self, global_seed: int, batch_id: int, hop: int):
        self.global_seed = global_seed
        self.batch_id = batch_id
        self.hop = hop
        self.key_prefix = hop_key_prefix(global_seed, batch_id, hop)

    def node_stream(self, dst_pos: int) -> CounterRng:
        return CounterRng(_fmix(self.key_prefix ^ dst_pos))


# ---------------------------------------------------------------------------
# configuration types (sampler.py:37-103)
# ---------------------------------------------------------------------------
@dataclass(frozen=True)
class SamplerVariant:
    map_impl: str = "flat_probing"
    set_impl: str = "vector_set"
    fuse: bool = True

    def __post_init__(self):
        if self.map_impl not in MAP_IMPLS:
            raise ValueError(f"unknown map_impl {self.map_impl!r}")
        if self.set_impl not in SET_IMPLS:
            raise ValueError(f"unknown set_impl {self.set_impl!r}")

    @property
    def descriptor(self) -> str:
        return "/".join((self.map_impl, self.set_impl, "fused" if self.fuse else "twopass"))

    @classmethod
    def from_descriptor(cls, desc: str) -> "SamplerVariant":
        parts = desc.split("/")
        if len(parts) != 3:
            raise ValueError(f"bad variant descriptor {desc!r}")
        if parts[2] not in ("fused", "twopass"):
            raise ValueError(f"bad fuse field in {desc!r}")
        return cls(parts[0], parts[1], parts[2] == "fused")


def list_variants() -> list[SamplerVariant]:
    return [SamplerVariant(m, s, f) for m, s, f in product(MAP_IMPLS, SET_IMPLS, (True, False))]


@dataclass(frozen=True)
class FanoutSpec:
    """Per-hop fanouts, outermost hop first (sampler.py:70-88)."""

    per_hop: tuple

    def __post_init__(self):
        if len(self.per_hop) < 1:
            raise ValueError("need at least one hop")
        if len(self.per_hop) > _lib.SAL_MAX_HOPS:
            raise ValueError(f"at most {_lib.SAL_MAX_HOPS} hops are supported")
        if any(int(d) < 0 for d in self.per_hop):
            raise ValueError("fanouts must be >= 0")
        object.__setattr__(self, "per_hop", tuple(int(d) for d in self.per_hop))

    def __len__(self):
        return len(self.per_hop)

    @classmethod
    def parse(cls, text: str) -> "FanoutSpec":
        return cls(tuple(int(t) for t in text.split(",")))


@dataclass(frozen=True)
class SeedBatch:
    batch_id: int
    dst_ids: np.ndarray

    def __post_init__(self):
        ids = np.ascontiguousarray(np.asarray(self.dst_ids, dtype=np.int64).reshape(-1))
        object.__setattr__(self, "dst_ids", ids)
        if len(np.unique(ids)) != len(ids):
            raise ValueError("seed IDs must be distinct")

    def __len__(self):
        return len(self.dst_ids)


def size_hint_for(seeds_len: int, fanouts: FanoutSpec, num_nodes: int) -> int:
    """Worst-case map size (sampler.py:321-325)."""
    est = seeds_len
    for d in reversed(fanouts.per_hop):
        est = min(num_nodes, est * (1 + d))
    return min(num_nodes, est)


# ---------------------------------------------------------------------------
# device id map (sampler.py:106-171)
# ---------------------------------------------------------------------------
def _pow2_at_least(n: int) -> int:
    return 1 << max(4, (int(n) - 1).bit_length())


class IdMap:
    """Insertion-ordered global<->local map held in HBM.

    table: open-addressing u64 slots {global:32 | local:32}; globals: int32
    local->global.  `size` is the host view, refreshed after each operation
    that changes it (one 8-byte read-back).
    """

    def __init__(self, variant: SamplerVariant = SamplerVariant(), size_hint: int | None = None,
                 device=None, *, _table=None, _globals=None, _size: int = 0):
        _lib.require_cuda()
        self.variant = variant
        self.device = torch.device(device or "cuda")
        if _table is not None:
            self._table, self._globals, self.size = _table, _globals, int(_size)
        else:
            cap = max(64, int(size_hint or 0))
            self._globals = torch.empty(cap, dtype=torch.int32, device=self.device)
            self._table = torch.empty(_pow2_at_least(2 * cap), dtype=torch.int64,
                                      device=self.device)
            self._table.fill_(-1)
            self.size = 0
        self._sizes = torch.zeros(2, dtype=torch.int64, device=self.device)

    @property
    def cstruct(self):
        return _lib.SalIdMap(self._table.data_ptr(), self._table.numel(),
                             self._globals.data_ptr(), self._globals.numel())

    def ensure_capacity(self, extra: int) -> None:
        need = self.size + int(extra)
        L = _lib.lib()
        if need > self._globals.numel():
            g = torch.empty(max(2 * self._globals.numel(), need), dtype=torch.int32,
                            device=self.device)
            g[:self.size] = self._globals[:self.size]
            self._globals = g
        if 2 * need > self._table.numel():
            self._table = torch.empty(_pow2_at_least(2 * need), dtype=torch.int64,
                                      device=self.device)
            c = self.cstruct
            _lib.check(L.sal_idmap_rehash(ctypes.byref(c), self.size, _lib.stream_ptr()),
                       "idmap_rehash")

    def insert(self, keys) -> None:
        """get-or-insert each key in order (insert_keys, _kernels.py:216-222)."""
        k = torch.from_numpy(np.ascontiguousarray(np.asarray(keys, dtype=np.int64).reshape(-1)))
        k = k.to(self.device)
        n = k.numel()
        if n == 0:
            return
        self.ensure_capacity(n)
        L = _lib.lib()
        scratch = torch.empty(3 * n, dtype=torch.int32, device=self.device)
        scan = torch.empty(L.sal_scan_ws_bytes(n), dtype=torch.uint8, device=self.device)
        nd = torch.empty(1, dtype=torch.int64, device=self.device)
        self._sizes[0] = self.size
        c = self.cstruct
        _lib.check(L.sal_idmap_insert(ctypes.byref(c), k.data_ptr(), n, self._sizes.data_ptr(),
                                      self._sizes[1:].data_ptr(), nd.data_ptr(),
                                      scratch.data_ptr(), scratch[n:].data_ptr(),
                                      scratch[2 * n:].data_ptr(), None, scan.data_ptr(),
                                      _lib.stream_ptr()), "idmap_insert")
        self.size = int(self._sizes[1].item())

    @property
    def global_ids(self) -> torch.Tensor:
        return self._globals[:self.size]

    def global_ids_host(self) -> np.ndarray:
        return self.global_ids.cpu().numpy().astype(np.int64)

    def global_of(self, local: int) -> int:
        if not 0 <= local < self.size:
            raise KeyError(local)
        return int(self._globals[local].item())

    def local_of(self, global_id: int) -> int:
        hit = torch.nonzero(self.global_ids == int(global_id))
        if hit.numel() == 0:
            raise KeyError(global_id)
        return int(hit[0, 0].item())

    def __len__(self):
        return self.size


# ---------------------------------------------------------------------------
# MFG types (sampler.py:178-235)
# ---------------------------------------------------------------------------
@dataclass(frozen=True)
class MfgLayer:
    """One bipartite hop: CSR-by-destination over local ids (device int32)."""

    num_dst: int
    num_src: int
    indptr: torch.Tensor     # int32 [num_dst + 1]
    src_local: torch.Tensor  # int32 [num_edges]

    @property
    def num_edges(self) -> int:
        return int(self.src_local.numel())

    def in_degree(self, dst_local: int) -> int:
        return int((self.indptr[dst_local + 1] - self.indptr[dst_local]).item())

    def to_host(self) -> dict:
        return dict(num_dst=self.num_dst, num_src=self.num_src,
                    indptr=self.indptr.cpu().numpy().astype(np.int64),
                    src_local=self.src_local.cpu().numpy().astype(np.int64))

    def structurally_equal(self, other) -> bool:
        a = self.to_host()
        b = other.to_host() if hasattr(other, "to_host") else dict(
            num_dst=other.num_dst, num_src=other.num_src, indptr=np.asarray(other.indptr),
            src_local=np.asarray(other.src_local))
        return (a["num_dst"] == b["num_dst"] and a["num_src"] == b["num_src"]
                and np.array_equal(a["indptr"], b["indptr"])
                and np.array_equal(a["src_local"], b["src_local"]))


@dataclass(frozen=True)
class Mfg:
    """Sampled multi-hop neighbourhood; layers[0] is the outermost hop."""

    layers: tuple
    id_map: IdMap
    seeds: SeedBatch
    workspace: object = None

    @property
    def num_nodes(self) -> int:
        return self.id_map.size

    @property
    def num_edges(self) -> int:
        return sum(l.num_edges for l in self.layers)

    def to_host(self):
        return self.id_map.global_ids_host(), [l.to_host() for l in self.layers]

    def digest(self) -> str:
        """blake2b-128 exactly as sampler.py:228-235 (int64 views)."""
        gids, layers = self.to_host()
        h = hashlib.blake2b(digest_size=16)
        h.update(np.ascontiguousarray(gids).tobytes())
        for l in layers:
            h.update(np.int64([l["num_dst"], l["num_src"]]).tobytes())
            h.update(np.ascontiguousarray(l["indptr"]).tobytes())
            h.update(np.ascontiguousarray(l["src_local"]).tobytes())
        return h.hexdigest()

    def structurally_equal(self, other: "Mfg") -> bool:
        return (len(self.layers) == len(other.layers)
                and torch.equal(self.id_map.global_ids, other.id_map.global_ids)
                and all(a.structurally_equal(b) for a, b in zip(self.layers, other.layers)))


# ---------------------------------------------------------------------------
# batch workspace: one in-flight multi-hop sample (sal_sample_mfg)
# ---------------------------------------------------------------------------
class MfgWorkspace:
    """Plan + layout + device bytes for one batch (worst-case capacities).

    Capacities follow size_hint_for: node_cap[h+1] = min(n, node_cap[h]*(1+f)),
    edge_cap[h] = node_cap[h]*f, so no hop ever needs a host round trip.
    """

    def __init__(self, num_nodes: int, fanouts: FanoutSpec, max_seeds: int, device=None,
                 last_hop_edges: bool = False, sample_lanes: int = 0, sample_bps: int = 0,
                 table_factor: int = 1, last_hop_fused: bool = False,
                 aggregate_bps: int = 0, reset_in_aggregate: bool = False,
                 resolve_in_aggregate: bool = False):
        """last_hop_edges: SAL_MFG_LAST_HOP_EDGES — the last hop only emits global
        source ids (src_glob); its relabel is skipped (training with the
        layer-0 mean read straight from the feature table).
        last_hop_fused: SAL_MFG_LAST_HOP_FUSED — run() builds hops 0..L-2 only and
        aggregate() samples the last hop straight into the layer-0 mean.
        aggregate_bps: resident blocks per SM of aggregate() (0 = as many as fit).
        reset_in_aggregate: (fused plans) run() skips the table/scan resets and
        aggregate() leaves them reset for the next batch; reset once here.
        resolve_in_aggregate: (fused plans) hop L-2's src_local is written by
        aggregate(), whose kernel runs that hop's relabel second pass (the fused
        kernel starts one launch earlier); read the MFG after aggregate()."""
        _lib.require_cuda()
        L = _lib.lib()
        self.device = torch.device(device or "cuda")
        self.fanouts = fanouts
        self.num_hops = len(fanouts)
        self.max_seeds = int(max_seeds)
        self.last_hop_fused = bool(last_hop_fused)
        self.last_hop_edges = bool(last_hop_edges) or self.last_hop_fused
        self.plan = _lib.SalMfgPlan()
        per = (ctypes.c_int32 * self.num_hops)(*fanouts.per_hop)
        flags = ((_lib.SAL_MFG_LAST_HOP_EDGES if self.last_hop_edges else 0)
                 | (_lib.SAL_MFG_LAST_HOP_FUSED if self.last_hop_fused else 0))
        _lib.check(L.sal_mfg_plan_init_ex(ctypes.byref(self.plan), self.num_hops, per,
                                          self.max_seeds, int(num_nodes), flags),
                   "mfg_plan_init")
        # design-space knobs (tools/sweep.py): sampler launch shape, id-table load
        if table_factor < 1 or table_factor & (table_factor - 1):
            raise ValueError("table_factor must be a power of two")
        self.plan.aggregate_blocks_per_sm = int(aggregate_bps)
        self.plan.reset_in_aggregate = 1 if (reset_in_aggregate and self.last_hop_fused) else 0
        self.plan.resolve_in_aggregate = 1 if (resolve_in_aggregate and self.last_hop_fused) else 0
        self.plan.sample_lanes = int(sample_lanes)
        self.plan.sample_blocks_per_sm = int(sample_bps)
        self.plan.table_cap = int(self.plan.table_cap) * int(table_factor)
        self.layout = _lib.SalMfgLayout()
        _lib.check(L.sal_mfg_layout_init(ctypes.byref(self.plan), ctypes.byref(self.layout)),
                   "mfg_layout_init")
        lay = self.layout
        self.buf = torch.empty(lay.total, dtype=torch.uint8, device=self.device)
        self.node_cap = [int(self.plan.node_cap[h]) for h in range(self.num_hops + 1)]
        self.edge_cap = [int(self.plan.edge_cap[h]) for h in range(self.num_hops)]
        self.globals = self._view(lay.globals, self.node_cap[-1], torch.int32)
        self.sizes = self._view(lay.sizes, self.num_hops + 1, torch.int64)
        self.etot = self._view(lay.etot, self.num_hops, torch.int64)
        self.table = self._view(lay.table, int(self.plan.table_cap), torch.int64)
        self.dst_indptr = [self._view(lay.dst_indptr[h], self.node_cap[h] + 1, torch.int32)
                           for h in range(self.num_hops)]
        self.src_local = [self._view(lay.src_local[h], self.edge_cap[h], torch.int32)
                          for h in range(self.num_hops)]
        # after a sample: global source ids of the LAST hop's edges (layer 0)
        self.src_glob = self._view(lay.src_glob, max(self.edge_cap + [1]), torch.int32)
        self.seeds = torch.empty(max(1, self.max_seeds), dtype=torch.int64, device=self.device)
        self.desc = torch.zeros(3, dtype=torch.int64, device=self.device)
        if self.plan.reset_in_aggregate:   # the first batch finds a reset table + scans
            self.reset_tables()

    def reset_tables(self) -> None:
        """Reset the id table and scan workspace (current stream): what a fused plan's
        aggregate() leaves behind, for a caller that ran run() without it."""
        lay = self.layout
        self.table.fill_(-1)
        self.buf[lay.scan:lay.scan + lay.scan_bytes].zero_()

    def _view(self, off: int, n: int, dt: torch.dtype) -> torch.Tensor:
        nbytes = n * torch.empty((), dtype=dt).element_size()
        return self.buf[off:off + nbytes].view(dt)

    def run(self, g: DeviceGraph, seeds_base: torch.Tensor, desc: torch.Tensor,
            global_seed: int, rng_policy: int = _lib.SAL_RNG_SPLITMIX, stream=None) -> None:
        """Enqueue the multi-hop sample on `stream` (no host sync)."""
        L = _lib.lib()
        gc = g.cstruct
        _lib.check(L.sal_sample_mfg(ctypes.byref(gc), ctypes.byref(self.plan),
                                    ctypes.byref(self.layout), self.buf.data_ptr(),
                                    seeds_base.data_ptr(), desc.data_ptr(),
                                    int(global_seed) & MASK64, int(rng_policy),
                                    _lib.stream_ptr(stream)), "sample_mfg")

    def run_next(self, g: DeviceGraph, seeds_base: torch.Tensor, desc_all: torch.Tensor,
                 n_steps: int, cursor: torch.Tensor, desc_out: torch.Tensor, global_seed: int,
                 rng_policy: int = _lib.SAL_RNG_SPLITMIX, stream=None) -> None:
        """run() on the next step of a device epoch plan: desc_out = desc_all[cursor]
        (an empty batch past n_steps), cursor += 1, then the sample — the cursor step
        rides in the seed-insertion kernel (sal_sample_mfg_next)."""
        L = _lib.lib()
        gc = g.cstruct
        _lib.check(L.sal_sample_mfg_next(ctypes.byref(gc), ctypes.byref(self.plan),
                                         ctypes.byref(self.layout), self.buf.data_ptr(),
                                         seeds_base.data_ptr(), desc_all.data_ptr(), int(n_steps),
                                         cursor.data_ptr(), desc_out.data_ptr(),
                                         int(global_seed) & MASK64, int(rng_policy),
                                         _lib.stream_ptr(stream)), "sample_mfg_next")

    def aggregate(self, g: DeviceGraph, table: torch.Tensor, out: torch.Tensor,
                  self_offset: int, desc: torch.Tensor, global_seed: int,
                  rng_policy: int = _lib.SAL_RNG_SPLITMIX, stream=None) -> None:
        """Fused last hop (after run(), same stream): out[d, :cols] = mean of the
        sampled table rows of layer-0 destination d, out[d, self_offset:+cols] =
        its own row (self_offset < 0: not written); cols = table.shape[1]."""
        if not self.last_hop_fused:
            raise ValueError("aggregate: workspace built without last_hop_fused")
        L = _lib.lib()
        gc = g.cstruct
        _lib.check(L.sal_sample_aggregate(
            ctypes.byref(gc), ctypes.byref(self.plan), ctypes.byref(self.layout),
            self.buf.data_ptr(), desc.data_ptr(), int(global_seed) & MASK64, int(rng_policy),
            table.data_ptr(), _lib.dtype_code(table.dtype), table.stride(0), table.shape[1],
            out.data_ptr(), _lib.dtype_code(out.dtype), out.stride(0), int(self_offset),
            _lib.stream_ptr(stream)), "sample_aggregate")

    def load_seeds(self, seeds: SeedBatch, stream=None) -> None:
        n = len(seeds)
        if n > self.max_seeds:
            raise ValueError(f"batch of {n} seeds exceeds workspace capacity {self.max_seeds}")
        s = stream or torch.cuda.current_stream()
        with torch.cuda.stream(s):
            if n:
                self.seeds[:n].copy_(torch.from_numpy(seeds.dst_ids), non_blocking=False)
            self.desc.copy_(torch.tensor([int(seeds.batch_id), 0, n], dtype=torch.int64))

    def read_extents(self):
        """One D2H: (sizes[L+1], etot[L]) as python ints (synchronises)."""
        both = torch.cat([self.sizes, self.etot]).cpu().tolist()
        return both[:self.num_hops + 1], both[self.num_hops + 1:]

    def to_mfg(self, seeds: SeedBatch, variant: SamplerVariant = SamplerVariant()) -> Mfg:
        if self.last_hop_edges:
            raise ValueError("to_mfg: the last hop of an edges-only workspace has no local ids")
        sizes, etot = self.read_extents()
        layers = []
        for h in range(self.num_hops):
            nd = sizes[h]
            layers.append(MfgLayer(num_dst=nd, num_src=sizes[h + 1],
                                   indptr=self.dst_indptr[h][:nd + 1],
                                   src_local=self.src_local[h][:etot[h]]))
        idm = IdMap(variant, device=self.device, _table=self.table, _globals=self.globals,
                    _size=sizes[-1])
        return Mfg(layers=tuple(reversed(layers)), id_map=idm, seeds=seeds, workspace=self)


# ---------------------------------------------------------------------------
# entry points (sampler.py:253-346)
# ---------------------------------------------------------------------------
def multihop_mfg(g, seeds: SeedBatch, fanouts: FanoutSpec, global_seed: int,
                 variant: SamplerVariant = SamplerVariant(), *, rng_policy: str = "splitmix",
                 stream=None) -> Mfg:
    """Expand seeds hop by hop on the GPU; hop h uses per_hop[L-1-h].

    Bit-identical to the reference (sampler.py:328-346) under the splitmix
    policy.  `rng_policy="philox"` selects the counter-based Philox stream.
    """
    dg = as_device_graph(g)
    ws = MfgWorkspace(dg.num_nodes, fanouts, len(seeds), device=dg.device)
    ws.load_seeds(seeds, stream)
    ws.run(dg, ws.seeds, ws.desc, global_seed, RNG_POLICIES[rng_policy], stream)
    return ws.to_mfg(seeds, variant)


def _hop(dg: DeviceGraph, id_map: IdMap, n_dst: int, fanout: int, key_prefix: int,
         policy: int = _lib.SAL_RNG_SPLITMIX, global_seed: int = 0, batch_id: int = 0,
         hop: int = 0, inject_pos: torch.Tensor | None = None, draws: torch.Tensor | None = None):
    """One hop against an arbitrary IdMap (the _run_hop path, sampler.py:284-300)."""
    L = _lib.lib()
    dev = id_map.device
    st = _lib.stream_ptr()
    nd = torch.tensor([n_dst], dtype=torch.int64, device=dev)
    dst_indptr = torch.empty(n_dst + 1, dtype=torch.int32, device=dev)
    etot = torch.empty(1, dtype=torch.int64, device=dev)
    scan = torch.empty(L.sal_scan_ws_bytes(max(n_dst, 1)), dtype=torch.uint8, device=dev)
    gc = dg.cstruct
    _lib.check(L.sal_hop_count(ctypes.byref(gc), id_map._globals.data_ptr(), nd.data_ptr(),
                               n_dst, fanout, dst_indptr.data_ptr(), etot.data_ptr(),
                               scan.data_ptr(), st), "hop_count")
    budget = int(etot.item())
    id_map.ensure_capacity(budget)
    e = max(budget, 1)
    src_glob = torch.empty(e, dtype=torch.int32, device=dev)
    slot = torch.empty(e, dtype=torch.int32, device=dev)
    rank = torch.empty(e, dtype=torch.int32, device=dev)
    src_local = torch.empty(budget, dtype=torch.int32, device=dev)
    c = id_map.cstruct
    _lib.check(L.sal_hop_sample(ctypes.byref(gc), ctypes.byref(c), nd.data_ptr(), n_dst, fanout,
                                key_prefix & MASK64, policy, global_seed & MASK64, batch_id, hop,
                                _lib.ptr(inject_pos), dst_indptr.data_ptr(), src_glob.data_ptr(),
                                slot.data_ptr(), _lib.ptr(draws), st), "hop_sample")
    sizes = id_map._sizes
    sizes[0] = id_map.size
    scan2 = torch.empty(L.sal_scan_ws_bytes(e), dtype=torch.uint8, device=dev)
    _lib.check(L.sal_hop_relabel(ctypes.byref(c), etot.data_ptr(), budget, sizes.data_ptr(),
                                 sizes[1:].data_ptr(), src_glob.data_ptr(), slot.data_ptr(),
                                 rank.data_ptr(), src_local.data_ptr(), scan2.data_ptr(), st),
               "hop_relabel")
    id_map.size = int(sizes[1].item())
    return MfgLayer(num_dst=n_dst, num_src=id_map.size, indptr=dst_indptr, src_local=src_local)


def one_hop_mfg(g, dst, d: int, rng: HopStream, variant: SamplerVariant, id_map: IdMap,
                *, inject_pos=None) -> MfgLayer:
    """Sample one hop; id_map must already hold the destinations as a prefix
    (sampler.py:303-318).  `inject_pos` (int64 per edge, hop_kernel pos_all
    layout) replays externally chosen slot positions instead of drawing."""
    dg = as_device_graph(g)
    if isinstance(dst, SeedBatch):
        n_dst = len(dst)
        pref = id_map.global_ids[:n_dst].cpu().numpy().astype(np.int64)
        if not np.array_equal(pref, dst.dst_ids):
            raise ValueError("id_map prefix does not match destination batch")
    else:
        n_dst = int(dst)
    if n_dst > id_map.size:
        raise ValueError("destination count exceeds id_map size")
    inj = None
    if inject_pos is not None:
        inj = torch.as_tensor(np.asarray(inject_pos, dtype=np.int64)).to(id_map.device)
    return _hop(dg, id_map, n_dst, int(d), rng.key_prefix, _lib.SAL_RNG_SPLITMIX,
                rng.global_seed, rng.batch_id, rng.hop, inj)


def sample_neighbors(g, v: int, d: int, rng: CounterRng) -> np.ndarray:
    """Edge-slot positions of node v sampled without replacement (sampler.py:253-273).

    Runs the device sampler on a one-destination hop whose neighbour list is
    replaced by slot positions; advances rng.counter by the draws consumed.  A
    stream already advanced to counter c continues exactly: draw k of the stream
    (key, c) is draw k of the fresh stream key + c * G (rng.py:38-51).
    """
    dg = as_device_graph(g)
    deg = dg.degree(int(v))
    dev = dg.device
    slots = DeviceGraph(1, torch.tensor([0, deg], dtype=torch.int64, device=dev),
                        torch.arange(max(deg, 1), dtype=torch.int32, device=dev)[:deg])
    idm = IdMap(device=dev, size_hint=1)
    idm.insert([0])
    draws = torch.zeros(1, dtype=torch.int32, device=dev)
    # key_0 = fmix(prefix ^ 0) must equal the continued key -> prefix = fmix^-1(key)
    key = (rng.key + rng.counter * _G) & MASK64
    layer = _hop(slots, idm, 1, int(d), _fmix_inverse(key), draws=draws)
    gids = idm.global_ids.cpu().numpy().astype(np.int64)
    rng.counter += int(draws.item())
    return gids[layer.src_local.cpu().numpy()]
