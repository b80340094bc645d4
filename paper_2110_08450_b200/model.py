"""GraphSAGE on device MFGs (PAPER.md:2562-2586 listing; mpnn.py layer rule).

SAGEConv-mean without bias:  h_dst' = W_neigh · mean_{src}(h) + W_self · h_dst,
then ReLU + dropout(0.5) between layers and log_softmax at the end.  The
mean is the library's CSR segment-reduce (forward and backward kernels); the
two products per layer are the only dense contractions and run as cuBLAS
GEMMs on the tensor cores (bf16 in the performance configuration, fp32 for
parity).

Static-shape mode: every layer can be given a padded destination count
(`n_pad`) with the true count read from device memory, so one training step
is a fixed sequence of kernels that CUDA graphs can capture.
"""

from __future__ import annotations

import math

import torch
import torch.nn as nn
import torch.nn.functional as F

from . import _lib


class SegmentMean(torch.autograd.Function):
    """out[d] = mean(h[src[e]] for e in row d); rows >= n_dst are zero."""

    @staticmethod
    def forward(ctx, h, indptr, src, n_pad, n_dst_dev, out_dtype):
        L = _lib.lib()
        out = torch.empty((n_pad, h.shape[1]), dtype=out_dtype, device=h.device)
        _lib.check(L.sal_segment_mean_fwd(indptr.data_ptr(), src.data_ptr(),
                                          _lib.ptr(n_dst_dev), n_pad, h.data_ptr(),
                                          _lib.dtype_code(h.dtype), h.stride(0), h.shape[1],
                                          out.data_ptr(), _lib.dtype_code(out_dtype),
                                          out.stride(0), _lib.stream_ptr()), "segment_mean_fwd")
        ctx.save_for_backward(indptr, src, n_dst_dev if n_dst_dev is not None else indptr)
        ctx.has_ndev = n_dst_dev is not None
        ctx.n_pad = n_pad
        ctx.h_shape = h.shape
        ctx.h_dtype = h.dtype
        return out

    @staticmethod
    def backward(ctx, g_out):
        if not ctx.needs_input_grad[0]:
            return None, None, None, None, None, None
        indptr, src, nd = ctx.saved_tensors
        L = _lib.lib()
        g_out = g_out.contiguous()
        g_h = torch.zeros(ctx.h_shape, dtype=torch.float32, device=g_out.device)
        _lib.check(L.sal_segment_mean_bwd(indptr.data_ptr(), src.data_ptr(),
                                          nd.data_ptr() if ctx.has_ndev else None, ctx.n_pad,
                                          g_out.data_ptr(), _lib.dtype_code(g_out.dtype),
                                          g_out.stride(0), g_out.shape[1], g_h.data_ptr(),
                                          g_h.stride(0), _lib.stream_ptr()), "segment_mean_bwd")
        if ctx.h_dtype != torch.float32:
            g_h = g_h.to(ctx.h_dtype)
        return g_h, None, None, None, None, None


class GlobalSegmentMean(torch.autograd.Function):
    """Layer-0 mean straight from the HBM feature table: X[globals[src[e]]]."""

    @staticmethod
    def forward(ctx, x, indptr, src, globals_, n_pad, n_dst_dev, out_dtype):
        L = _lib.lib()
        out = torch.empty((n_pad, x.shape[1]), dtype=out_dtype, device=x.device)
        _lib.check(L.sal_segment_mean_fwd_global(indptr.data_ptr(), src.data_ptr(),
                                                 globals_.data_ptr(), _lib.ptr(n_dst_dev),
                                                 n_pad, x.data_ptr(), _lib.dtype_code(x.dtype),
                                                 x.stride(0), x.shape[1], out.data_ptr(),
                                                 _lib.dtype_code(out_dtype), out.stride(0),
                                                 _lib.stream_ptr()), "segment_mean_fwd_global")
        return out

    @staticmethod
    def backward(ctx, g):
        return None, None, None, None, None, None, None


class SAGEConv(nn.Module):
    """Mean SAGEConv, bias=False (PyG semantics used by PAPER.md:2563-2575)."""

    def __init__(self, f_in: int, f_out: int):
        super().__init__()
        self.w_neigh = nn.Parameter(torch.empty(f_out, f_in))
        self.w_self = nn.Parameter(torch.empty(f_out, f_in))
        self.reset_parameters()

    def reset_parameters(self):
        bound = 1.0 / math.sqrt(self.w_self.shape[1])
        nn.init.uniform_(self.w_neigh, -bound, bound)
        nn.init.uniform_(self.w_self, -bound, bound)

    def forward(self, mean: torch.Tensor, h_dst: torch.Tensor) -> torch.Tensor:
        return F.linear(mean, self.w_neigh.to(mean.dtype)) + \
            F.linear(h_dst, self.w_self.to(h_dst.dtype))


class GraphSAGE(nn.Module):
    """3-layer GraphSAGE of the paper (hidden 256 at papers100M shape)."""

    def __init__(self, f_in: int, hidden: int, num_classes: int, num_layers: int = 3,
                 dropout: float = 0.5):
        super().__init__()
        dims = [f_in] + [hidden] * (num_layers - 1) + [num_classes]
        self.convs = nn.ModuleList(SAGEConv(a, b) for a, b in zip(dims[:-1], dims[1:]))
        self.dropout = dropout

    def forward(self, x: torch.Tensor, adjs, act_dtype: torch.dtype = torch.float32,
                x_global: tuple | None = None) -> torch.Tensor:
        """adjs: per layer (indptr int32, src int32, n_dst_pad, n_dst_dev or None).

        x holds the layer-0 source rows in local order.  With `x_global =
        (table, globals)` layer 0 aggregates straight from the feature table
        and x only needs the destination rows.
        """
        h = x
        n = len(self.convs)
        for i, (conv, (indptr, src, n_pad, n_dev)) in enumerate(zip(self.convs, adjs)):
            if i == 0 and x_global is not None:
                table, gl = x_global
                mean = GlobalSegmentMean.apply(table, indptr, src, gl, n_pad, n_dev, act_dtype)
            else:
                mean = SegmentMean.apply(h, indptr, src, n_pad, n_dev, act_dtype)
            h_dst = h[:n_pad]
            if h_dst.dtype != act_dtype:
                h_dst = h_dst.to(act_dtype)
            h = conv(mean, h_dst)
            if i != n - 1:
                h = F.relu(h)
                if self.dropout and self.training:
                    h = F.dropout(h, p=self.dropout, training=True)
        return torch.log_softmax(h.float(), dim=-1)
