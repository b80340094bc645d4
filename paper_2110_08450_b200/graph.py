"""Graph / feature / label storage: host types and the HBM-resident replica.

Host side mirrors the reference's L0 data store (graph.py:39-303 of
mfgprep): `CsrGraph`, `FeatureMatrix`, `LabelVector`, `from_edge_list`,
`synth_graph`, `generate_features`, `generate_labels`.  These are fixture
builders (numpy), not part of the hot path; `synth_graph` reproduces the
reference's generator stream exactly so both sides can be fed identical
inputs (pinned by tests/test_host.py against the reference's checksums).

`DeviceGraph` is the B200 layout every kernel reads:
    indptr   int64[n+1]          (1.6e9 slots at papers100M shape)
    indices  int32[E]            (node ids < 2^31)
    features fp16/fp32 [n, f_pad] rows padded to a 16-byte stride
    labels   int64[n]
One full replica per GPU (~36 GB at papers100M shape of 180 GB HBM).
`synth_graph_device` builds the same law directly in HBM.
"""

from __future__ import annotations

import zlib
import struct
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib

DTYPE_F16 = 1
DTYPE_F32 = 2


@dataclass(frozen=True)
class CsrGraph:
    """Host CSR adjacency (graph.py:39-85); neighbors keep insertion order."""

    num_nodes: int
    indptr: np.ndarray
    indices: np.ndarray

    @property
    def num_edges(self) -> int:
        return len(self.indices)

    def degree(self, v: int) -> int:
        return int(self.indptr[v + 1] - self.indptr[v])

    def neighbors(self, v: int) -> np.ndarray:
        return self.indices[self.indptr[v]:self.indptr[v + 1]]

    def degrees(self) -> np.ndarray:
        return np.diff(self.indptr)

    def max_degree(self) -> int:
        return int(self.degrees().max()) if self.num_nodes else 0

    def validate(self) -> None:
        if self.indptr[0] != 0 or self.indptr[-1] != self.num_edges:
            raise ValueError("indptr endpoints inconsistent with edge count")
        if np.any(np.diff(self.indptr) < 0):
            raise ValueError("indptr must be non-decreasing")
        if self.num_edges and (self.indices.min() < 0 or self.indices.max() >= self.num_nodes):
            raise ValueError("neighbor ID out of range")

    def checksum(self) -> int:
        """crc32 over (indptr int64, indices int64, num_nodes) (graph.py:78-85)."""
        h = zlib.crc32(np.ascontiguousarray(self.indptr, dtype=np.int64).tobytes())
        h = zlib.crc32(np.ascontiguousarray(self.indices, dtype=np.int64).tobytes(), h)
        return zlib.crc32(struct.pack("<Q", self.num_nodes), h)


@dataclass(frozen=True)
class FeatureMatrix:
    """Row-major node features, f16 or f32 (graph.py:88-104)."""

    rows: int
    cols: int
    data: np.ndarray

    def __post_init__(self):
        if self.data.dtype not in (np.float16, np.float32):
            raise ValueError("feature dtype must be float16 or float32")
        if self.data.shape != (self.rows, self.cols):
            raise ValueError("feature data shape mismatch")

    @property
    def dtype_code(self) -> int:
        return DTYPE_F16 if self.data.dtype == np.float16 else DTYPE_F32


@dataclass(frozen=True)
class LabelVector:
    values: np.ndarray
    num_classes: int

    def __post_init__(self):
        if len(self.values) and (self.values.min() < 0 or self.values.max() >= self.num_classes):
            raise ValueError("label out of range")


def from_edge_list(edges, num_nodes: int, make_undirected: bool = False) -> CsrGraph:
    """CSR from (src, dst) pairs in input order (graph.py:134-162 semantics).

    Undirected input contributes (s,d) then (d,s) for each pair, so every
    row lists its slots in edge-sequence order.  Counting sort, O(E).
    """
    arr = np.asarray(edges if isinstance(edges, np.ndarray) else list(edges), dtype=np.int64)
    arr = arr.reshape(-1, 2)
    src, dst = arr[:, 0], arr[:, 1]
    bad = np.flatnonzero((src < 0) | (src >= num_nodes) | (dst < 0) | (dst >= num_nodes))
    if bad.size:
        i = int(bad[0])
        raise ValueError(f"edge {i} = ({src[i]}, {dst[i]}) has endpoint outside [0, {num_nodes})")
    if make_undirected:
        s2 = np.empty(2 * len(src), dtype=np.int64)
        d2 = np.empty_like(s2)
        s2[0::2], s2[1::2] = src, dst
        d2[0::2], d2[1::2] = dst, src
        src, dst = s2, d2
    counts = np.bincount(src, minlength=num_nodes)
    indptr = np.zeros(num_nodes + 1, dtype=np.int64)
    np.cumsum(counts, out=indptr[1:])
    order = np.argsort(src, kind="stable")
    g = CsrGraph(num_nodes=num_nodes, indptr=indptr, indices=dst[order])
    g.validate()
    return g


def synth_graph(n: int, avg_degree: float, exponent: float = 3.0, seed: int = 0) -> CsrGraph:
    """Pareto configuration-model multigraph (law of graph.py:252-280).

    Uses the same numpy Generator call sequence as the reference so that,
    for equal arguments, the graphs are identical (same checksum).
    """
    if n < 1:
        raise ValueError("n must be >= 1")
    if avg_degree < 0:
        raise ValueError("avg_degree must be >= 0")
    rng = np.random.default_rng(seed)
    if np.isfinite(exponent):
        if exponent <= 2.0:
            raise ValueError("exponent must be > 2 for a finite mean degree")
        shape = exponent - 1.0
        degs = np.rint(avg_degree * (shape - 1.0) / shape
                       * (1.0 + rng.pareto(shape, size=n))).astype(np.int64)
        degs = np.clip(degs, 0, n - 1)
    else:
        degs = np.full(n, int(round(avg_degree)), dtype=np.int64)
    if int(degs.sum()) % 2:
        degs[int(rng.integers(n))] += 1
    stubs = np.repeat(np.arange(n, dtype=np.int64), degs)
    rng.shuffle(stubs)
    return from_edge_list(stubs.reshape(-1, 2), n, make_undirected=True)


def generate_features(n: int, f: int, dtype: str = "f32", seed: int = 0) -> FeatureMatrix:
    """uniform [-1, 1] f32, optionally rounded to f16 (graph.py:283-292 law)."""
    if dtype not in ("f16", "f32"):
        raise ValueError(f"unknown feature dtype {dtype!r}")
    data = np.random.default_rng(seed).uniform(-1.0, 1.0, size=(n, f)).astype(np.float32)
    return FeatureMatrix(rows=n, cols=f, data=data.astype(np.float16) if dtype == "f16" else data)


def generate_labels(n: int, num_classes: int, seed: int = 0) -> LabelVector:
    """i.i.d. uniform classes (graph.py:295-298 law)."""
    vals = np.random.default_rng(seed).integers(0, num_classes, size=n, dtype=np.int64)
    return LabelVector(values=vals, num_classes=num_classes)


def planted_labels(features: np.ndarray, num_classes: int, seed: int = 0) -> LabelVector:
    """Learnable labels: argmax of a fixed random projection of the features.

    The reference's labels carry no signal (graph.py:295-298); the accuracy
    check of the north star needs a label that a GraphSAGE model can learn.
    """
    rng = np.random.default_rng(seed)
    proj = rng.standard_normal((features.shape[1], num_classes)).astype(np.float32)
    vals = np.argmax(np.asarray(features, dtype=np.float32) @ proj, axis=1).astype(np.int64)
    return LabelVector(values=vals, num_classes=num_classes)


# ---------------------------------------------------------------------------
# HBM-resident replica
# ---------------------------------------------------------------------------
def _pad_cols(f: int, elem_bytes: int) -> int:
    """Row stride (elements) of an HBM feature table: a 16-byte multiple, and for 16-bit
    tables of 65..127 columns a full 256 B row — whole 32 B sectors and all 16 lanes of
    the row kernels, and the width the model reads anyway (train._model_width).
    Products' 100 fp16 columns: fused last hop 69.4 -> 57.5 us, epoch 0.031 -> 0.029 s
    against the 104-column (208 B) stride (profiles/r2_ab_pad128.txt)."""
    if elem_bytes == 2 and 64 < f < 128:
        return 128
    per = 16 // elem_bytes
    return (f + per - 1) // per * per


class DeviceGraph:
    """CSR graph (+ optional features / labels) resident in one GPU's HBM."""

    def __init__(self, num_nodes: int, indptr: torch.Tensor, indices: torch.Tensor,
                 features: torch.Tensor | None = None, num_features: int | None = None,
                 labels: torch.Tensor | None = None, num_classes: int = 0):
        if num_nodes >= 2**31 - 1:
            raise ValueError("device graphs are limited to 2^31-1 nodes")
        self.num_nodes = int(num_nodes)
        self.indptr = indptr
        self.indices = indices
        self.features = features          # [n, f_pad] (padded row stride)
        self.num_features = num_features if num_features is not None else (
            features.shape[1] if features is not None else 0)
        self.labels = labels
        self.num_classes = num_classes
        self.device = indptr.device
        self._max_degree = None
        self._c = _lib.SalGraph(self.num_nodes, int(indices.numel()), indptr.data_ptr(),
                                indices.data_ptr())

    @property
    def num_edges(self) -> int:
        return int(self.indices.numel())

    @property
    def cstruct(self):
        return self._c

    def max_degree(self) -> int:
        if self._max_degree is None:
            self._max_degree = int((self.indptr[1:] - self.indptr[:-1]).max().item()) \
                if self.num_nodes else 0
        return self._max_degree

    def degree(self, v: int) -> int:
        return int((self.indptr[v + 1] - self.indptr[v]).item())

    def feature_view(self) -> torch.Tensor:
        """[n, f] view (stride = padded row)."""
        return self.features[:, :self.num_features]

    @classmethod
    def from_host(cls, g, fm: FeatureMatrix | None = None, y: LabelVector | None = None,
                  device=None) -> "DeviceGraph":
        """Upload a host CsrGraph (reference or ours) + features + labels."""
        _lib.require_cuda()
        dev = torch.device(device or "cuda")
        indptr = torch.from_numpy(np.ascontiguousarray(g.indptr, dtype=np.int64)).to(dev)
        idx = np.asarray(g.indices)
        if len(idx) and int(idx.max()) >= 2**31:
            raise ValueError("node ids must fit in int32")
        indices = torch.from_numpy(np.ascontiguousarray(idx, dtype=np.int32)).to(dev)
        feats = None
        nf = None
        if fm is not None:
            data = np.asarray(fm.data)
            tdt = torch.float16 if data.dtype == np.float16 else torch.float32
            nf = data.shape[1]
            fpad = _pad_cols(nf, data.dtype.itemsize)
            feats = torch.zeros((data.shape[0], fpad), dtype=tdt, device=dev)
            feats[:, :nf] = torch.from_numpy(np.ascontiguousarray(data)).to(dev)
        labels = None
        nc = 0
        if y is not None:
            labels = torch.from_numpy(np.ascontiguousarray(y.values, dtype=np.int64)).to(dev)
            nc = int(y.num_classes)
        return cls(int(g.num_nodes), indptr, indices, feats, nf, labels, nc)


def as_device_graph(g, fm=None, y=None) -> DeviceGraph:
    """Accept a DeviceGraph or upload (and cache on the host object) a host graph."""
    if isinstance(g, DeviceGraph):
        return g
    cache = _UPLOAD_CACHE.get(id(g))
    if cache is not None and cache[0] is g:
        dg = cache[1]
    else:
        dg = DeviceGraph.from_host(g)
        _UPLOAD_CACHE[id(g)] = (g, dg)
    return dg


_UPLOAD_CACHE: dict = {}


def upload_features(fm: FeatureMatrix, device=None) -> torch.Tensor:
    """Feature table in HBM with a 16-byte padded row stride; returns [n, f] view."""
    key = id(fm)
    hit = _FEAT_CACHE.get(key)
    if hit is not None and hit[0] is fm:
        return hit[1]
    data = np.asarray(fm.data)
    tdt = torch.float16 if data.dtype == np.float16 else torch.float32
    fpad = _pad_cols(data.shape[1], data.dtype.itemsize)
    t = torch.zeros((data.shape[0], fpad), dtype=tdt, device=device or "cuda")
    t[:, :data.shape[1]] = torch.from_numpy(np.ascontiguousarray(data)).to(t.device)
    view = t[:, :data.shape[1]]
    _FEAT_CACHE[key] = (fm, view)
    return view


_FEAT_CACHE: dict = {}


def upload_labels(y: LabelVector, device=None) -> torch.Tensor:
    key = id(y)
    hit = _LAB_CACHE.get(key)
    if hit is not None and hit[0] is y:
        return hit[1]
    t = torch.from_numpy(np.ascontiguousarray(y.values, dtype=np.int64)).to(device or "cuda")
    _LAB_CACHE[key] = (y, t)
    return t


_LAB_CACHE: dict = {}


def synth_odd_fix_node(n: int, seed: int) -> int:
    """The node whose degree absorbs an odd stub total (graph.py:273-274 law):
    a counter-based pick, so the host restatement (oracle.synth_graph_host) agrees."""
    z = (int(seed) ^ 0x0DD5EED) & (2**64 - 1)
    z = (z + 0x9E3779B97F4A7C15) & (2**64 - 1)
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & (2**64 - 1)
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & (2**64 - 1)
    z ^= z >> 31
    return int(z % n)


def synth_graph_device(n: int, avg_degree: float, exponent: float = 3.0, seed: int = 0,
                       num_features: int = 0, num_classes: int = 0, feature_seed: int = 1,
                       label_seed: int = 1, device=None) -> DeviceGraph:
    """Build a synth_graph-law graph (+ fp16 features, labels) directly in HBM.

    Degrees: rint(scale * (1 - u)^(-1/a)) clipped to [0, n-1] with u a
    counter-based (Philox) uniform per node (sal_gen_degrees); an odd stub
    total adds one stub at synth_odd_fix_node; stubs paired by the library's
    Feistel matching; features uniform [-1, 1) -> fp16; labels uniform.  Every
    step is counter-based and exactly rounded, so oracle.synth_graph_host
    rebuilds the same arrays on the host (tests/test_gpu_generate.py).  Peak
    extra memory is one int32 owner array of E entries.
    """
    _lib.require_cuda()
    if n < 1:
        raise ValueError("n must be >= 1")
    if avg_degree < 0:
        raise ValueError("avg_degree must be >= 0")
    L = _lib.lib()
    dev = torch.device(device or "cuda")
    st = _lib.stream_ptr()
    if np.isfinite(exponent):
        if exponent <= 2.0:
            raise ValueError("exponent must be > 2 for a finite mean degree")
        a = exponent - 1.0
        scale = avg_degree * (a - 1.0) / a
        degs = torch.empty(n, dtype=torch.int64, device=dev)
        _lib.check(L.sal_gen_degrees(n, int(seed) & (2**64 - 1), scale, a, degs.data_ptr(), st),
                   "gen_degrees")
    else:
        degs = torch.full((n,), int(round(avg_degree)), dtype=torch.int64, device=dev)
    total = int(degs.sum().item())
    if total % 2:
        degs[synth_odd_fix_node(n, seed)] += 1
        total += 1
    indptr = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    torch.cumsum(degs, 0, out=indptr[1:])
    del degs
    owner = torch.empty(total, dtype=torch.int32, device=dev)
    _lib.check(L.sal_gen_owner(indptr.data_ptr(), n, owner.data_ptr(), st), "gen_owner")
    indices = torch.empty(total, dtype=torch.int32, device=dev)
    _lib.check(L.sal_gen_pairing(owner.data_ptr(), total, int(seed) & (2**64 - 1),
                                 indices.data_ptr(), st), "gen_pairing")
    del owner
    feats = None
    if num_features:
        fpad = _pad_cols(num_features, 2)
        feats = torch.empty((n, fpad), dtype=torch.float16, device=dev)
        if fpad != num_features:
            feats[:, num_features:].zero_()
        _lib.check(L.sal_gen_features_uniform(n, num_features, fpad, int(feature_seed),
                                              feats.data_ptr(), st), "gen_features")
    labels = None
    if num_classes:
        labels = torch.empty(n, dtype=torch.int64, device=dev)
        _lib.check(L.sal_gen_labels_uniform(n, num_classes, int(label_seed), labels.data_ptr(),
                                            st), "gen_labels")
    return DeviceGraph(n, indptr, indices, feats, num_features or None, labels, num_classes)
