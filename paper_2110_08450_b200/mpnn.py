"""Mean-aggregation MPNN evaluated on the GPU (drop-in for mfgprep.mpnn).

Layer rule (mpnn.py:1-14 of the reference): h_dst = W_self h_dst +
W_neigh mean(h_src over sampled in-neighbours), empty mean = 0, no bias, no
activation, fp32.  The mean is the library's segment-reduce kernel
(sal_segment_mean_fwd); the two products are plain fp32 GEMMs with TF32
disabled, so results match the reference to ~1e-6.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .sampler import Mfg


@dataclass(frozen=True)
class LayerWeights:
    w_self: np.ndarray   # (f_out, f_in)
    w_neigh: np.ndarray  # (f_out, f_in)

    def __post_init__(self):
        if np.shape(self.w_self) != np.shape(self.w_neigh):
            raise ValueError("weight shape mismatch")


def init_weights(f_in: int, f_hidden: int, num_layers: int, seed: int = 0) -> list[LayerWeights]:
    """uniform(-0.1, 0.1) weights, same numpy stream as mpnn.py:34-45."""
    rng = np.random.default_rng(seed)
    dims = [f_in] + [f_hidden] * num_layers
    ws = []
    for d_in, d_out in zip(dims[:-1], dims[1:]):
        a = rng.uniform(-0.1, 0.1, size=(d_out, d_in)).astype(np.float32)
        b = rng.uniform(-0.1, 0.1, size=(d_out, d_in)).astype(np.float32)
        ws.append(LayerWeights(w_self=a, w_neigh=b))
    return ws


def segment_mean(indptr: torch.Tensor, src: torch.Tensor, h: torch.Tensor, num_dst: int,
                 out_dtype: torch.dtype = torch.float32, n_pad: int | None = None,
                 n_dst_dev: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """out[d] = mean(h[src[indptr[d]:indptr[d+1]]]) through sal_segment_mean_fwd."""
    rows = num_dst if n_pad is None else n_pad
    out = torch.empty((rows, h.shape[1]), dtype=out_dtype, device=h.device)
    L = _lib.lib()
    _lib.check(L.sal_segment_mean_fwd(indptr.data_ptr(), src.data_ptr(), _lib.ptr(n_dst_dev),
                                      rows, h.data_ptr(), _lib.dtype_code(h.dtype), h.stride(0),
                                      h.shape[1], out.data_ptr(), _lib.dtype_code(out_dtype),
                                      out.stride(0), _lib.stream_ptr(stream)),
               "segment_mean_fwd")
    return out


def _check_dims(cols: int, weights) -> None:
    d = cols
    for i, w in enumerate(weights):
        if np.shape(w.w_self)[1] != d:
            raise ValueError(f"layer {i} expects input dim {np.shape(w.w_self)[1]}, got {d}")
        d = np.shape(w.w_self)[0]


def _as_dev(w, dev):
    return torch.as_tensor(np.asarray(w, dtype=np.float32)).to(dev)


def mfg_forward(mfg: Mfg, features, weights) -> torch.Tensor:
    """Evaluate over local ids (mpnn.py:68-83); returns |seeds| rows on device."""
    if len(weights) != len(mfg.layers):
        raise ValueError("one weight set per MFG layer required")
    dev = mfg.id_map.device
    h = torch.as_tensor(features).to(dev)
    if h.dtype != torch.float32:
        h = h.float()
    if h.shape[0] != mfg.num_nodes:
        raise ValueError("feature rows must cover the whole id_map")
    _check_dims(h.shape[1], weights)
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        for layer, w in zip(mfg.layers, weights):
            neigh = segment_mean(layer.indptr, layer.src_local, h, layer.num_dst)
            h = h[:layer.num_dst] @ _as_dev(w.w_self, dev).T + neigh @ _as_dev(w.w_neigh, dev).T
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev
    return h


def sampled_reference_forward(mfg: Mfg, features_global, weights) -> torch.Tensor:
    """Same math as mfg_forward, indexing the GLOBAL feature matrix (mpnn.py:86-111).

    Layer 0 never touches a sliced local buffer: every edge is resolved to its global
    endpoint through the id map and the row is read from the global table on the
    device (sal_segment_mean_fwd_global), the destinations' own rows likewise; the
    layers above index hidden rows by local id (the reference's dict keyed by global
    id is the same bijection).  A disagreement with mfg_forward pinpoints a local-id
    or slicing defect.  Returns |seeds| rows on device."""
    if len(weights) != len(mfg.layers):
        raise ValueError("one weight set per MFG layer required")
    dev = mfg.id_map.device
    X = torch.as_tensor(features_global).to(dev)
    if X.dtype != torch.float32:
        X = X.float()
    X = X.contiguous()
    _check_dims(X.shape[1], weights)
    gids = mfg.id_map.global_ids
    L = _lib.lib()
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        h = None
        for i, (layer, w) in enumerate(zip(mfg.layers, weights)):
            if i == 0:
                neigh = torch.empty((layer.num_dst, X.shape[1]), dtype=torch.float32, device=dev)
                if layer.num_dst:
                    _lib.check(L.sal_segment_mean_fwd_global(
                        layer.indptr.data_ptr(), layer.src_local.data_ptr(), gids.data_ptr(),
                        None, layer.num_dst, X.data_ptr(), _lib.SAL_F32, X.stride(0),
                        X.shape[1], neigh.data_ptr(), _lib.SAL_F32, neigh.stride(0),
                        _lib.stream_ptr()), "segment_mean_fwd_global")
                h_dst = X[gids[:layer.num_dst].long()]
            else:
                neigh = segment_mean(layer.indptr, layer.src_local, h, layer.num_dst)
                h_dst = h[:layer.num_dst]
            h = h_dst @ _as_dev(w.w_self, dev).T + neigh @ _as_dev(w.w_neigh, dev).T
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev
    return h


def full_forward(g, X, weights, dst_ids, num_layers: int | None = None) -> torch.Tensor:
    """Exact full-neighbourhood evaluation (mpnn.py:114-135) on the device graph."""
    from .graph import as_device_graph
    dg = as_device_graph(g)
    if num_layers is None:
        num_layers = len(weights)
    if num_layers < 1:
        raise ValueError("need at least one layer")
    if dg.num_edges >= 2**31:
        raise ValueError("full_forward needs < 2^31 edges (int32 row pointer)")
    dev = dg.device
    h = torch.as_tensor(np.asarray(X, dtype=np.float32)).to(dev)
    _check_dims(h.shape[1], weights)
    indptr32 = dg.indptr.to(torch.int32)
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        for w in weights[:num_layers]:
            neigh = segment_mean(indptr32, dg.indices, h, dg.num_nodes)
            h = h @ _as_dev(w.w_self, dev).T + neigh @ _as_dev(w.w_neigh, dev).T
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev
    return h[torch.as_tensor(np.asarray(dst_ids, dtype=np.int64)).to(dev)]
