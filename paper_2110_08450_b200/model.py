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


# ---------------------------------------------------------------------------
# Explicit-backward GraphSAGE for the training hot path
# ---------------------------------------------------------------------------
class FusedSAGE:
    """GraphSAGE with a hand-scheduled forward/backward (no autograd graph).

    Parameters live in one flat fp32 buffer (Adam updates it with one fused
    kernel); a bf16 shadow copy feeds the tensor-core GEMMs and is refreshed
    with one cast after each optimizer step.  Weight gradients are written
    straight into the flat fp32 gradient buffer by cuBLAS (bf16 x bf16 ->
    fp32 output), so there is no gradient zeroing or accumulation pass, and
    the flat buffer is what the data-parallel all-reduce sends.

    Per layer i (consumption order):
        mean_i = segment_mean(h_i)                         (library kernel)
        z_i    = h_i[:n_pad_i] @ Ws_i^T + mean_i @ Wn_i^T  (2 cuBLAS GEMMs)
        h_i+1  = relu_dropout(z_i)                         (library kernel)
    loss = lsm_nll(z_L-1, labels)  (fused log_softmax + NLL + gradient)
    """

    def __init__(self, f_in: int, hidden: int, num_classes: int, num_layers: int = 3,
                 dropout: float = 0.5, device=None, seed: int = 0,
                 act_dtype: torch.dtype = torch.bfloat16):
        dev = torch.device(device or "cuda")
        self.dims = [f_in] + [hidden] * (num_layers - 1) + [num_classes]
        self.L = num_layers
        self.p = float(dropout)
        self.act = act_dtype
        shapes = []
        for a, b in zip(self.dims[:-1], self.dims[1:]):
            shapes += [(b, a), (b, a)]   # (w_neigh, w_self) per layer
        total = sum(r * c for r, c in shapes)
        self.flat = torch.empty(total, dtype=torch.float32, device=dev)
        self.grad = torch.zeros(total, dtype=torch.float32, device=dev)
        self.shadow = torch.empty(total, dtype=act_dtype, device=dev)
        g = torch.Generator(device="cpu")
        g.manual_seed(seed)
        off = 0
        self.w, self.g, self.wb = [], [], []
        for r, c in shapes:
            bound = 1.0 / math.sqrt(c)
            self.flat[off:off + r * c] = (torch.rand(r * c, generator=g) * 2 - 1).mul_(bound).to(dev)
            self.w.append(self.flat[off:off + r * c].view(r, c))
            self.g.append(self.grad[off:off + r * c].view(r, c))
            self.wb.append(self.shadow[off:off + r * c].view(r, c))
            off += r * c
        self.param = torch.nn.Parameter(self.flat, requires_grad=False)
        self.param.grad = self.grad
        self.refresh_shadow()
        self.training = True
        self.seed = seed

    def refresh_shadow(self):
        self.shadow.copy_(self.flat)

    def state_dict(self):
        return {"flat": self.flat.detach().clone(), "dims": list(self.dims)}

    def load_weights(self, layer_weights):
        """layer_weights: list of (w_self, w_neigh) arrays/tensors (out, in)."""
        for i, (ws, wn) in enumerate(layer_weights):
            self.w[2 * i].copy_(torch.as_tensor(wn, dtype=torch.float32))
            self.w[2 * i + 1].copy_(torch.as_tensor(ws, dtype=torch.float32))
        self.refresh_shadow()

    # ---------------------------------------------------------------- fwd
    def forward(self, x: torch.Tensor, adjs, x_global=None, salt: torch.Tensor | None = None):
        """Returns (logits, saved) — saved holds what backward needs."""
        L = _lib.lib()
        st = _lib.stream_ptr()
        h = x
        saved = []
        for i in range(self.L):
            indptr, src, n_pad, n_dev = adjs[i]
            f = h.shape[1] if not (i == 0 and x_global is not None) else x_global[0].shape[1]
            mean = torch.empty((n_pad, f), dtype=self.act, device=h.device)
            if i == 0 and x_global is not None:
                table, gl = x_global
                _lib.check(L.sal_segment_mean_fwd_global(
                    indptr.data_ptr(), src.data_ptr(), gl.data_ptr(), _lib.ptr(n_dev), n_pad,
                    table.data_ptr(), _lib.dtype_code(table.dtype), table.stride(0), f,
                    mean.data_ptr(), _lib.dtype_code(self.act), mean.stride(0), st),
                    "segment_mean_fwd_global")
            else:
                _lib.check(L.sal_segment_mean_fwd(
                    indptr.data_ptr(), src.data_ptr(), _lib.ptr(n_dev), n_pad, h.data_ptr(),
                    _lib.dtype_code(h.dtype), h.stride(0), f, mean.data_ptr(),
                    _lib.dtype_code(self.act), mean.stride(0), st), "segment_mean_fwd")
            h_dst = h[:n_pad]
            z = torch.mm(h_dst, self.wb[2 * i + 1].t())
            z.addmm_(mean, self.wb[2 * i].t())
            rec = dict(h=h, mean=mean, n_pad=n_pad, adj=adjs[i])
            if i != self.L - 1:
                y = torch.empty_like(z)
                mask = torch.empty(z.numel() // 8, dtype=torch.uint8, device=z.device)
                p = self.p if self.training else 0.0
                _lib.check(L.sal_relu_dropout_fwd(
                    z.data_ptr(), y.data_ptr(), mask.data_ptr(), z.numel(),
                    _lib.dtype_code(z.dtype), p, (self.seed * 1000003 + i) & (2**64 - 1),
                    _lib.ptr(salt), st), "relu_dropout_fwd")
                rec["mask"] = mask
                h = y
            else:
                h = z
            saved.append(rec)
        return h, saved

    def loss(self, logits: torch.Tensor, labels: torch.Tensor):
        """Fused log_softmax + NLL; returns (loss scalar fp32, dlogits)."""
        L = _lib.lib()
        loss = torch.zeros((), dtype=torch.float32, device=logits.device)
        dlog = torch.empty_like(logits)
        rows = min(logits.shape[0], labels.shape[0])
        _lib.check(L.sal_lsm_nll(logits.data_ptr(), logits.stride(0), rows, logits.shape[1],
                                 _lib.dtype_code(logits.dtype), labels.data_ptr(),
                                 loss.data_ptr(), dlog.data_ptr(), dlog.stride(0),
                                 _lib.stream_ptr()), "lsm_nll")
        return loss, dlog

    # ---------------------------------------------------------------- bwd
    def backward(self, dlogits: torch.Tensor, saved) -> None:
        """Writes every weight gradient into self.grad (overwrite semantics)."""
        L = _lib.lib()
        st = _lib.stream_ptr()
        dz = dlogits
        for i in reversed(range(self.L)):
            rec = saved[i]
            h, mean, n_pad = rec["h"], rec["mean"], rec["n_pad"]
            dzt = dz.t()
            _mm_f32(dzt, mean, self.g[2 * i])
            _mm_f32(dzt, h[:n_pad], self.g[2 * i + 1])
            if i == 0:
                break
            # input gradient of layer i: self term + scatter of the mean term
            dh = torch.zeros((h.shape[0], h.shape[1]), dtype=torch.float32, device=h.device)
            _mm_f32(dz, self.wb[2 * i + 1], dh[:n_pad])
            dmean = torch.mm(dz, self.wb[2 * i])
            indptr, src, _, n_dev = rec["adj"]
            _lib.check(L.sal_segment_mean_bwd(
                indptr.data_ptr(), src.data_ptr(), _lib.ptr(n_dev), n_pad, dmean.data_ptr(),
                _lib.dtype_code(dmean.dtype), dmean.stride(0), dmean.shape[1], dh.data_ptr(),
                dh.stride(0), st), "segment_mean_bwd")
            # through relu+dropout of the previous layer's output
            prev_mask = saved[i - 1]["mask"]
            dzp = torch.empty((h.shape[0], h.shape[1]), dtype=self.act, device=h.device)
            _lib.check(L.sal_relu_dropout_bwd(
                dh.data_ptr(), _lib.SAL_F32, prev_mask.data_ptr(), dzp.data_ptr(),
                _lib.dtype_code(self.act), dh.numel(), self.p if self.training else 0.0, st),
                "relu_dropout_bwd")
            dz = dzp

    @torch.no_grad()
    def predict(self, x, adjs, x_global=None):
        was = self.training
        self.training = False
        try:
            logits, _ = self.forward(x, adjs, x_global)
        finally:
            self.training = was
        return logits


def _mm_f32(a: torch.Tensor, b: torch.Tensor, out: torch.Tensor) -> None:
    """out (fp32) = a @ b; 16-bit operands accumulate and store in fp32 (cuBLAS)."""
    if a.dtype == torch.float32:
        torch.mm(a, b, out=out)
    else:
        torch.mm(a, b, out_dtype=torch.float32, out=out)
