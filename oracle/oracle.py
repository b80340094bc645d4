"""Python face of the CPU oracle (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may
import this module — as the checker or as the timed CPU baseline, never as
the product path.  It wraps oracle/liboracle.so (a C restatement of the
reference's numba kernels) and adds numpy restatements of the pieces the
reference itself writes in numpy (mpnn.py mean aggregation / forward).

Every function cites the reference file:line it restates
(/root/reference/pkg/src/mfgprep).  Pinned by tests/test_oracle.py against
golden vectors produced by the reference (tests/golden/make_golden.py).
"""

from __future__ import annotations

import ctypes
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "liboracle.so"

_i64p = ctypes.POINTER(ctypes.c_int64)
_i32p = ctypes.POINTER(ctypes.c_int32)
_u64p = ctypes.POINTER(ctypes.c_uint64)

MASK64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15


def build() -> Path:
    """Compile liboracle.so with the committed Makefile."""
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB_PATH


_LIB = None


def lib():
    global _LIB
    if _LIB is None:
        if not LIB_PATH.exists():
            build()
        L = ctypes.CDLL(str(LIB_PATH))
        L.orc_mix64.restype = ctypes.c_uint64
        L.orc_mix64.argtypes = [ctypes.c_uint64]
        L.orc_hop_prefix.restype = ctypes.c_uint64
        L.orc_hop_prefix.argtypes = [ctypes.c_uint64] * 3
        L.orc_sample_positions.restype = ctypes.c_int64
        L.orc_sample_positions.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64, _i64p]
        L.orc_multihop.restype = ctypes.c_int64
        L.orc_multihop.argtypes = [_i64p, _i32p, ctypes.c_int64, _i64p, ctypes.c_int64, _i32p,
                                   ctypes.c_int, ctypes.c_uint64, ctypes.c_int64, _i64p,
                                   ctypes.c_int64, _i64p, ctypes.c_int64, _i64p, ctypes.c_int64,
                                   _i64p]
        L.orc_gather_f16.restype = None
        L.orc_gather_f16.argtypes = [ctypes.c_void_p, ctypes.c_int64, _i64p, ctypes.c_int64,
                                     ctypes.c_void_p]
        L.orc_gather_f32.restype = None
        L.orc_gather_f32.argtypes = [ctypes.c_void_p, ctypes.c_int64, _i64p, ctypes.c_int64,
                                     ctypes.c_void_p]
        L.orc_epoch_prep.restype = ctypes.c_double
        L.orc_epoch_prep.argtypes = [_i64p, _i32p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int,
                                     ctypes.c_int64, _i64p, _i64p, _i64p, _i64p, ctypes.c_int64,
                                     _i32p, ctypes.c_int, ctypes.c_uint64, ctypes.c_int, _i64p,
                                     _u64p]
        L.orc_synth_degrees.restype = None
        L.orc_synth_degrees.argtypes = [ctypes.c_int64, ctypes.c_uint64, ctypes.c_double,
                                        ctypes.c_double, _i64p, ctypes.c_int]
        L.orc_synth_pairing.restype = ctypes.c_int
        L.orc_synth_pairing.argtypes = [_i64p, ctypes.c_int64, ctypes.c_uint64, _i32p, ctypes.c_int]
        L.orc_synth_features.restype = None
        L.orc_synth_features.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_int32,
                                         ctypes.c_int64, ctypes.c_uint64, ctypes.c_void_p,
                                         ctypes.c_int]
        L.orc_synth_labels.restype = None
        L.orc_synth_labels.argtypes = [ctypes.c_int64, ctypes.c_int32, ctypes.c_uint64, _i64p,
                                       ctypes.c_int]
        L.orc_f32_to_f16.restype = ctypes.c_uint16
        L.orc_f32_to_f16.argtypes = [ctypes.c_float]
        _LIB = L
    return _LIB


def _p(a, t):
    return a.ctypes.data_as(t)


# --------------------------------------------------------------------------
# RNG (rng.py:16-35, sampler.py:238-250)
# --------------------------------------------------------------------------
def mix64(z: int) -> int:
    return int(lib().orc_mix64(z & MASK64))


def hop_prefix(seed: int, batch: int, hop: int) -> int:
    return int(lib().orc_hop_prefix(seed & MASK64, batch & MASK64, hop & MASK64))


def stream_key(seed: int, batch: int, hop: int, pos: int) -> int:
    """rng.py:24-30"""
    return mix64(hop_prefix(seed, batch, hop) ^ pos)


def sample_positions(key: int, deg: int, d: int) -> list[int]:
    """_kernels.py:102-147 / reference.py:21-34"""
    out = np.empty(max(1, min(deg, d) if deg > d else deg), dtype=np.int64)
    n = lib().orc_sample_positions(key & MASK64, deg, d, _p(out, _i64p))
    return out[:n].tolist()


# --------------------------------------------------------------------------
# multi-hop MFG (sampler.py:328-346)
# --------------------------------------------------------------------------
def node_caps(nseeds: int, per_hop, num_nodes: int):
    caps = [min(nseeds, num_nodes)]
    edges = []
    for f in reversed(per_hop):
        edges.append(caps[-1] * f)
        caps.append(max(caps[-1], min(num_nodes, caps[-1] * (1 + f))))
    return caps, edges


def multihop(indptr, indices, num_nodes, seeds, per_hop, global_seed, batch_id):
    """Returns (global_ids, layers) with layers in consumption order, each
    a dict(num_dst, num_src, indptr int64, src_local int64)."""
    indptr = np.ascontiguousarray(indptr, dtype=np.int64)
    indices = np.ascontiguousarray(indices, dtype=np.int32)
    seeds = np.ascontiguousarray(seeds, dtype=np.int64)
    per = np.ascontiguousarray(per_hop, dtype=np.int32)
    L = len(per)
    caps, edges = node_caps(len(seeds), list(per_hop), num_nodes)
    gcap = max(1, caps[-1])
    scap = max(1, sum(edges))
    dcap = sum(c + 1 for c in caps[:-1])
    g = np.empty(gcap, dtype=np.int64)
    s = np.empty(scap, dtype=np.int64)
    d = np.empty(dcap, dtype=np.int64)
    meta = np.empty(3 * L, dtype=np.int64)
    n = lib().orc_multihop(_p(indptr, _i64p), _p(indices, _i32p), num_nodes, _p(seeds, _i64p),
                           len(seeds), _p(per, _i32p), L, global_seed & MASK64, batch_id,
                           _p(g, _i64p), gcap, _p(s, _i64p), scap, _p(d, _i64p), dcap,
                           _p(meta, _i64p))
    if n < 0:
        raise RuntimeError("oracle multihop overflow")
    layers = []
    so = do = 0
    for h in range(L):
        nd, ns, ne = (int(x) for x in meta[3 * h:3 * h + 3])
        layers.append(dict(num_dst=nd, num_src=ns, indptr=d[do:do + nd + 1].copy(),
                           src_local=s[so:so + ne].copy()))
        so += ne
        do += nd + 1
    return g[:n].copy(), list(reversed(layers))


def gather_features(data: np.ndarray, ids) -> np.ndarray:
    """slice_features (prep.py:153-171) -> gather_f16/gather_f32 (_kernels.py:225-252)."""
    ids = np.ascontiguousarray(ids, dtype=np.int64)
    data = np.ascontiguousarray(data)
    out = np.empty((len(ids), data.shape[1]), dtype=np.float32)
    if len(ids) == 0:
        return out
    if data.dtype == np.float16:
        lib().orc_gather_f16(data.ctypes.data, data.shape[1], _p(ids, _i64p), len(ids),
                             out.ctypes.data)
    elif data.dtype == np.float32:
        lib().orc_gather_f32(data.ctypes.data, data.shape[1], _p(ids, _i64p), len(ids),
                             out.ctypes.data)
    else:
        raise ValueError("feature dtype must be float16 or float32")
    return out


def gather_labels(values, ids) -> np.ndarray:
    """slice_labels (prep.py:174-182)."""
    return np.asarray(values, dtype=np.int64)[np.asarray(ids, dtype=np.int64)]


def mfg_digest(global_ids, layers) -> str:
    """Mfg.digest (sampler.py:228-235)."""
    import hashlib
    h = hashlib.blake2b(digest_size=16)
    h.update(np.ascontiguousarray(global_ids, dtype=np.int64).tobytes())
    for l in layers:
        h.update(np.int64([l["num_dst"], l["num_src"]]).tobytes())
        h.update(np.ascontiguousarray(l["indptr"], dtype=np.int64).tobytes())
        h.update(np.ascontiguousarray(l["src_local"], dtype=np.int64).tobytes())
    return h.hexdigest()


def batch_digest(mfg_hex: str, features: np.ndarray, labels: np.ndarray) -> str:
    """PreparedBatch.digest (prep.py:132-137)."""
    import hashlib
    h = hashlib.blake2b(digest_size=16)
    h.update(mfg_hex.encode())
    h.update(np.ascontiguousarray(features, dtype=np.float32).tobytes())
    h.update(np.ascontiguousarray(labels, dtype=np.int64).tobytes())
    return h.hexdigest()


# --------------------------------------------------------------------------
# aggregation (mpnn.py:57-83), numpy
# --------------------------------------------------------------------------
def mean_neighbors(h, indptr, src_local, num_dst) -> np.ndarray:
    """mpnn.py:57-65: f32 sum in edge order, / in-degree, 0 when empty."""
    h = np.asarray(h, dtype=np.float32)
    acc = np.zeros((num_dst, h.shape[1]), dtype=np.float32)
    deg = np.diff(np.asarray(indptr, dtype=np.int64))
    dst = np.repeat(np.arange(num_dst), deg)
    np.add.at(acc, dst, h[np.asarray(src_local, dtype=np.int64)])
    nz = deg > 0
    acc[nz] /= deg[nz].astype(np.float32)[:, None]
    return acc


def mfg_forward(layers, features, weights) -> np.ndarray:
    """mpnn.py:68-83 (weights: list of (w_self, w_neigh), shape (out, in))."""
    h = np.asarray(features, dtype=np.float32)
    for lay, (ws, wn) in zip(layers, weights):
        neigh = mean_neighbors(h, lay["indptr"], lay["src_local"], lay["num_dst"])
        h = h[:lay["num_dst"]] @ np.asarray(ws, np.float32).T + neigh @ np.asarray(wn, np.float32).T
    return h


# --------------------------------------------------------------------------
# epoch prep (prep.py:226-341) — the timed CPU baseline
# --------------------------------------------------------------------------
def epoch_prep(indptr, indices, num_nodes, features, labels, batches, per_hop, global_seed,
               nthreads: int):
    """Prepare every batch of `batches` (list of (batch_id, seeds)) with
    `nthreads` workers.  Returns (wall_s, stats[nb,4], checksums)."""
    indptr = np.ascontiguousarray(indptr, dtype=np.int64)
    indices = np.ascontiguousarray(indices, dtype=np.int32)
    feats = np.ascontiguousarray(features)
    is16 = 1 if feats.dtype == np.float16 else 0
    if not is16 and feats.dtype != np.float32:
        raise ValueError("feature dtype must be float16 or float32")
    lab = None if labels is None else np.ascontiguousarray(labels, dtype=np.int64)
    ids = np.asarray([b for b, _ in batches], dtype=np.int64)
    offs = np.zeros(len(batches) + 1, dtype=np.int64)
    offs[1:] = np.cumsum([len(s) for _, s in batches])
    seeds = (np.concatenate([np.asarray(s, dtype=np.int64) for _, s in batches])
             if batches else np.zeros(1, dtype=np.int64))
    per = np.ascontiguousarray(per_hop, dtype=np.int32)
    stats = np.zeros((len(batches), 4), dtype=np.int64)
    ck = np.zeros(max(1, len(batches)), dtype=np.uint64)
    wall = lib().orc_epoch_prep(
        _p(indptr, _i64p), _p(indices, _i32p), num_nodes, feats.ctypes.data, is16,
        feats.shape[1], None if lab is None else _p(lab, _i64p), _p(seeds, _i64p),
        _p(offs, _i64p), _p(ids, _i64p), len(batches), _p(per, _i32p), len(per),
        global_seed & MASK64, nthreads, _p(stats, _i64p), _p(ck, _u64p))
    return wall, stats, ck


# --------------------------------------------------------------------------
# synthetic inputs: host restatement of the device generator
# (paper_2110_08450_b200/csrc/generate.cu; law of graph.py:252-298)
# --------------------------------------------------------------------------
def _odd_fix_node(n: int, seed: int) -> int:
    """graph.synth_odd_fix_node (counter-based pick of graph.py:273-274)."""
    return int(mix64(((int(seed) ^ 0x0DD5EED) + GOLDEN) & MASK64) % n)


def synth_degrees(n: int, avg_degree: float, exponent: float, seed: int, nthreads: int = 8):
    a = exponent - 1.0
    scale = avg_degree * (a - 1.0) / a
    degs = np.empty(n, dtype=np.int64)
    lib().orc_synth_degrees(n, int(seed) & MASK64, scale, a, _p(degs, _i64p), nthreads)
    return degs


def synth_graph_host(n: int, avg_degree: float, exponent: float = 3.0, seed: int = 0,
                     num_features: int = 0, num_classes: int = 0, feature_seed: int = 1,
                     label_seed: int = 1, nthreads: int = 8, feature_stride: int | None = None):
    """The arrays graph.synth_graph_device builds, rebuilt on the host: returns
    dict(indptr int64 [n+1], indices int32 [E], features fp16 [n, stride] or
    None, labels int64 [n] or None)."""
    if np.isfinite(exponent):
        degs = synth_degrees(n, avg_degree, exponent, seed, nthreads)
    else:
        degs = np.full(n, int(round(avg_degree)), dtype=np.int64)
    if int(degs.sum()) % 2:
        degs[_odd_fix_node(n, seed)] += 1
    indptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(degs, out=indptr[1:])
    del degs
    indices = np.empty(max(int(indptr[-1]), 1), dtype=np.int32)[:int(indptr[-1])]
    rc = lib().orc_synth_pairing(_p(indptr, _i64p), n, int(seed) & MASK64, _p(indices, _i32p),
                                 nthreads)
    if rc != 0:
        raise RuntimeError(f"orc_synth_pairing failed ({rc})")
    feats = None
    if num_features:
        stride = feature_stride or -(-num_features // 8) * 8
        feats = np.zeros((n, stride), dtype=np.float16)
        lib().orc_synth_features(0, n, num_features, stride, int(feature_seed) & MASK64,
                                 feats.ctypes.data, nthreads)
    labels = None
    if num_classes:
        labels = np.empty(n, dtype=np.int64)
        lib().orc_synth_labels(n, num_classes, int(label_seed) & MASK64, _p(labels, _i64p),
                               nthreads)
    return dict(indptr=indptr, indices=indices, features=feats, labels=labels)


def f32_to_f16_bits(x: float) -> int:
    return int(lib().orc_f32_to_f16(x))
