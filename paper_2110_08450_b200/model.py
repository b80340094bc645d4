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

    Activations use the library's "cat" layout: the input of layer i is a
    [rows, 2f] buffer with h_i in the right half; segment_mean writes mean_i
    into the left half of the first n_pad (destination) rows, so each
    SAGEConv is ONE tensor-core GEMM  z = [mean | h_dst] @ [W_neigh | W_self]^T
    and its backward is one weight-gradient GEMM (bf16 x bf16 -> fp32 straight
    into the flat gradient buffer) plus, above layer 0, one input-gradient
    GEMM dA = dz @ W_cat followed by sal_mean_bwd_t, which gathers the
    mean-term gradient per source row over the reverse adjacency and applies
    the ReLU/dropout backward in the same pass.

    Parameters: one flat fp32 buffer (per layer [f_out, 2 f_in] = [W_n | W_s]),
    updated by one fused Adam kernel that also refreshes the bf16 shadow the
    GEMMs read.
    """

    def __init__(self, f_in: int, hidden: int, num_classes: int, num_layers: int = 3,
                 dropout: float = 0.5, device=None, seed: int = 0,
                 act_dtype: torch.dtype = torch.bfloat16, lr: float = 0.003,
                 betas=(0.9, 0.999), eps: float = 1e-8):
        dev = torch.device(device or "cuda")
        self.device = dev
        self.dims = [f_in] + [hidden] * (num_layers - 1) + [num_classes]
        self.L = num_layers
        self.p = float(dropout)
        self.act = act_dtype
        self.lr, self.betas, self.eps = lr, betas, eps
        # the output layer's rows are padded to a multiple of 16 (zero weights, zero
        # gradients): every logits / dlogits row is 16-byte aligned and the tcgen05
        # GEMMs take c_pad as their N (output layer) or K (its input gradient)
        self.c_pad = -(-num_classes // 16) * 16
        rows_pad = self.dims[1:-1] + [self.c_pad]
        shapes = [(r, 2 * a) for a, r in zip(self.dims[:-1], rows_pad)]
        total = sum(r * c for r, c in shapes)
        self.flat = torch.zeros(total, dtype=torch.float32, device=dev)
        self.grad = torch.zeros(total, dtype=torch.float32, device=dev)
        self.m = torch.zeros(total, dtype=torch.float32, device=dev)
        self.v = torch.zeros(total, dtype=torch.float32, device=dev)
        self.t = torch.zeros(1, dtype=torch.int64, device=dev)
        self.shadow = torch.empty(total, dtype=act_dtype, device=dev)
        g = torch.Generator(device="cpu")
        g.manual_seed(seed)
        off = 0
        # w/g: logical [f_out, 2 f_in] views; wb/gp: the padded views the GEMMs use
        self.w, self.g, self.wb, self.gp = [], [], [], []
        for (r, c), fo in zip(shapes, self.dims[1:]):
            bound = 1.0 / math.sqrt(c // 2)   # SAGEConv-style U(-1/sqrt(f_in), 1/sqrt(f_in))
            self.flat[off:off + fo * c] = ((torch.rand(fo * c, generator=g) * 2 - 1)
                                           * bound).to(dev)
            self.w.append(self.flat[off:off + r * c].view(r, c)[:fo])
            self.gp.append(self.grad[off:off + r * c].view(r, c))
            self.g.append(self.gp[-1][:fo])
            self.wb.append(self.shadow[off:off + r * c].view(r, c))
            off += r * c
        self._dlog = None
        self.refresh_shadow()
        self.training = True
        self.seed = seed
        self.use_tc = True
        # K = 2 f_in of the layers on the tcgen05 forward
        self.tc_fwd_k = (256, 512)
        # tcgen05 weight gradients (tiled split-K, sal_tc_sage_wgrad) where the
        # shapes allow; cuBLAS for the rest
        self.tc_wgrad = True
        # the output layer on tcgen05 (sal_tc_sage_head: logits in TMEM, loss, dlogits,
        # dA and dW in one kernel): 179.9 against 179.6 us per step for cuBLAS x3 +
        # lsm_nll, three launches fewer
        self.tc_head = True
        # the hidden layers' input-gradient GEMM dA = dz @ W_cat on tcgen05
        # (sal_tc_gemm_nn): alone 6.8 against 4.5 us for cuBLAS at [6144 x 256] @
        # [256 x 512], but in the overlapped step (fused last hop beside the backward)
        # 149 against 156.5 us per step (tools/step_ab.py): no library GEMM in the step
        self.tc_dA = True
        # weight gradients of the layers above 0 on a second stream, beside the
        # input-gradient chain
        self.overlap_wgrad = True   # measured 0.233 -> 0.228 s per papers epoch
        # fork each overlapped weight gradient after the layer's dA GEMM (True) or
        # before it (False)
        self.wgrad_fork_late = True
        # the last input gradient writes only the rows layer 0's weight gradient reads
        self.mbt_live = True
        # input gradients as sal_mean_bwd: single-in-edge rows destination-major (each
        # dA row read once for all its sources), the rest source-major (bit-identical
        # to sal_mean_bwd_t)
        self.mbt_split = True
        # zero-fill the padding rows of the tcgen05 forward's output and mask in training
        self.pad_fill = False
        self._wgrad_stream = torch.cuda.Stream(device=dev)

    # ------------------------------------------------------------- weights
    def refresh_shadow(self):
        self.shadow.copy_(self.flat)

    def w_neigh(self, i):
        return self.w[i][:, :self.dims[i]]

    def w_self(self, i):
        return self.w[i][:, self.dims[i]:]

    def load_weights(self, layer_weights):
        """layer_weights: list of (w_self, w_neigh) arrays/tensors (out, in)."""
        for i, (ws, wn) in enumerate(layer_weights):
            self.w_neigh(i).copy_(torch.as_tensor(wn, dtype=torch.float32))
            self.w_self(i).copy_(torch.as_tensor(ws, dtype=torch.float32))
        self.refresh_shadow()

    def adam_step(self):
        L = _lib.lib()
        _lib.check(L.sal_adam_step(self.flat.data_ptr(), self.grad.data_ptr(), self.m.data_ptr(),
                                   self.v.data_ptr(),
                                   self.shadow.data_ptr() if self.act == torch.bfloat16 else None,
                                   self.flat.numel(), self.lr, self.betas[0], self.betas[1],
                                   self.eps, self.t.data_ptr(), 0, _lib.stream_ptr()),
                   "adam_step")
        if self.act != torch.bfloat16:
            self.refresh_shadow()

    def optimizer_tensors(self):
        return [self.flat, self.m, self.v, self.t]

    def _tc_layer(self, i: int) -> bool:
        """Layers the hand-written tcgen05 forward covers: bf16, K = 2 f_in = 256 or
        512, N = f_out = 256, with a hidden layer after it (the ReLU/dropout
        epilogue)."""
        return (self.use_tc and self.act == torch.bfloat16 and i != self.L - 1
                and 2 * self.dims[i] in self.tc_fwd_k and self.dims[i + 1] == 256)

    def _tc_wgrad_layer(self, i: int) -> bool:
        """dW_i on sal_tc_sage_wgrad: bf16 operands, dW rows a multiple of 16 (the
        output layer's c_pad rows included), cols a multiple of 128."""
        return (self.tc_wgrad and self.act == torch.bfloat16
                and self.gp[i].shape[0] % 16 == 0 and self.gp[i].shape[1] % 128 == 0)

    def _tc_dA_layer(self, i: int) -> bool:
        """dA_i = dz_i @ W_cat_i on sal_tc_gemm_nn: K = rows of W_cat (f_out or c_pad)
        a multiple of 16, N = 2 f_in a multiple of 128."""
        return (self.tc_dA and self.act == torch.bfloat16
                and self.wb[i].shape[0] % 16 == 0 and self.wb[i].shape[1] % 128 == 0)

    # ------------------------------------------------------------- buffers
    def cat_input(self, x: torch.Tensor) -> torch.Tensor:
        """Copy a plain [N, f] layer-0 input into a fresh cat buffer [N, 2 f_in]
        (f <= f_in; columns past f stay zero)."""
        fm = self.dims[0]
        a = torch.zeros((x.shape[0], 2 * fm), dtype=self.act, device=x.device)
        a[:, fm:fm + x.shape[1]] = x
        return a

    # ------------------------------------------------------------- fwd
    def forward(self, a0: torch.Tensor, adjs, x_global=None, salt: torch.Tensor | None = None,
                head: bool = False, mean0_ready: bool = False):
        """a0: layer-0 cat buffer (right half = features in local order).

        adjs[i] = (indptr, src, n_pad, n_dst_dev).  With x_global = (table,
        edge_global_ids) layer 0's mean is read straight from the feature table
        (the sampler's per-edge global ids of the last hop).
        head: stop after the output layer's mean (loss_backward runs the rest).
        mean0_ready: a0's left half already holds layer 0's mean (the fused last hop,
        sal_sample_aggregate).
        Returns (logits [n_pad_last, C] or None with head, saved)."""
        L = _lib.lib()
        st = _lib.stream_ptr()
        a = a0
        saved = []
        for i in range(self.L):
            indptr, src, n_pad, n_dev = adjs[i]
            f = self.dims[i]
            h = a[:, f:]
            mean = a[:n_pad, :f]
            if i == 0 and mean0_ready:
                pass
            elif i == 0 and x_global is not None:
                # gather-free layer 0: edges carry global ids, rows come from the table
                table, gsrc = x_global
                # the table may be narrower than the model's (zero-padded) input width.
                # Padding rows are left as they are: the layer-0 buffers start zeroed and
                # only ever hold finite values, the tcgen05 forward reads them only inside
                # the last partial tile and the weight gradient pairs them with zero dz
                # (451 K padded vs 175 K real rows at the (20,20,20) inference shape)
                _lib.check(L.sal_segment_mean_fwd_ex(
                    indptr.data_ptr(), gsrc.data_ptr(), _lib.ptr(n_dev), n_pad,
                    table.data_ptr(), _lib.dtype_code(table.dtype), table.stride(0),
                    min(f, table.shape[1]), mean.data_ptr(), _lib.dtype_code(self.act),
                    a.stride(0), _lib.SAL_SEG_NO_PAD_FILL if n_dev is not None else 0, st),
                    "segment_mean_fwd(table)")
            else:
                _lib.check(L.sal_segment_mean_fwd(
                    indptr.data_ptr(), src.data_ptr(), _lib.ptr(n_dev), n_pad, h.data_ptr(),
                    _lib.dtype_code(h.dtype), a.stride(0), f, mean.data_ptr(),
                    _lib.dtype_code(self.act), a.stride(0), st), "segment_mean_fwd")
            rec = dict(a=a, n_pad=n_pad, adj=adjs[i])
            if i != self.L - 1:
                fo = self.dims[i + 1]
                nxt = torch.empty((n_pad, 2 * fo), dtype=self.act, device=a.device)
                mask = torch.empty(n_pad * fo // 8, dtype=torch.uint8, device=a.device)
                p = self.p if self.training else 0.0
                seed = (self.seed * 1000003 + i) & (2**64 - 1)
                if self._tc_layer(i):
                    # tcgen05 GEMM with the ReLU/dropout epilogue: z never reaches HBM
                    _lib.check(L.sal_tc_sage_fwd(
                        a.data_ptr(), a.stride(0), n_pad, _lib.ptr(n_dev), self.wb[i].data_ptr(),
                        fo, 2 * f,
                        nxt[:, fo:].data_ptr(), nxt.stride(0), mask.data_ptr(), p, seed,
                        # padding rows (past the true count) are left unwritten unless
                        # pad_fill: no kernel reads them (the next layer's mean and GEMMs
                        # touch only live rows, and mean_bwd_t's sum for a padding row is 0
                        # whatever its mask bits)
                        _lib.ptr(salt), 1 if (self.training and self.pad_fill) else 3, st),
                        "tc_sage_fwd")
                else:
                    z = torch.mm(a[:n_pad], self.wb[i].t())
                    _lib.check(L.sal_relu_dropout_fwd(
                        z.data_ptr(), z.stride(0), nxt[:, fo:].data_ptr(), nxt.stride(0), n_pad,
                        fo, _lib.dtype_code(self.act), mask.data_ptr(), p, seed, _lib.ptr(salt),
                        st), "relu_dropout_fwd")
                rec["mask"] = mask
                a = nxt
            elif head:  # the fused output layer (loss_backward) computes the logits
                a = None
            else:
                a = torch.mm(a[:n_pad], self.wb[i].t())[:, :self.dims[-1]]
            saved.append(rec)
        return a, saved

    def loss(self, logits: torch.Tensor, labels: torch.Tensor, out: torch.Tensor | None = None,
             zeroed: bool = False):
        """Fused log_softmax + NLL; returns (loss scalar fp32, dlogits [rows, c_pad]).

        dlogits lives in a persistent buffer whose padded columns stay zero.
        zeroed: `out` is already zero (the trainer's step_tail clears it)."""
        L = _lib.lib()
        loss = out if out is not None else torch.empty((), dtype=torch.float32,
                                                       device=logits.device)
        if not (zeroed and out is not None):
            loss.zero_()
        n = logits.shape[0]
        if self._dlog is None or self._dlog.shape[0] != n or self._dlog.dtype != logits.dtype:
            self._dlog = torch.zeros((n, self.c_pad), dtype=logits.dtype, device=logits.device)
        dlog = self._dlog
        rows = min(logits.shape[0], labels.shape[0])
        _lib.check(L.sal_lsm_nll(logits.data_ptr(), logits.stride(0), rows, logits.shape[1],
                                 _lib.dtype_code(logits.dtype), labels.data_ptr(),
                                 loss.data_ptr(), dlog.data_ptr(), dlog.stride(0),
                                 _lib.stream_ptr()), "lsm_nll")
        return loss, dlog

    # ------------------------------------------------------------- bwd
    def tc_grad_spans(self):
        """(pointer, bytes) of the gradient blocks the split-K tcgen05 weight
        gradient accumulates into; a caller that zeroes them off the critical path
        passes grads_zeroed=True to backward()."""
        return [(self.gp[i].data_ptr(), self.gp[i].numel() * 4) for i in range(self.L)
                if self._tc_wgrad_layer(i) or (i == self.L - 1 and self.head_ok())]

    def backward(self, dlogits: torch.Tensor, saved, transposes=None,
                 grads_zeroed: bool = False, t_events=None) -> None:
        """Writes every weight gradient into self.grad (overwrite semantics; with
        grads_zeroed the tcgen05 layers accumulate into blocks the caller zeroed).

        transposes[i] = (tindptr, tdst) reverse adjacency of layer i (i >= 1);
        built here when not supplied (the trainer builds them on the prep
        stream).  t_events[i]: an event the current stream waits on before it reads
        transposes[i]."""
        self._backward_below(self.L - 1, dlogits, saved, transposes, grads_zeroed, t_events)

    def _backward_below(self, top: int, dz, saved, transposes, grads_zeroed: bool,
                        t_events=None):
        """Weight gradients of layers top..0 from dz of layer top, and the input
        gradients between them."""
        cs = torch.cuda.current_stream()
        ws = self._wgrad_stream if self.overlap_wgrad else None
        forked = False

        def fork_wgrad(i: int, dz) -> None:
            # the weight gradient of layer i only reads dz_i: it runs on a second
            # stream beside the input-gradient chain (dA GEMM -> mean_bwd_t)
            ws.wait_stream(cs)
            with torch.cuda.stream(ws):
                self._wgrad(i, dz, saved, grads_zeroed)
            dz.record_stream(ws)

        for i in reversed(range(top + 1)):
            # fork after the dA GEMM (wgrad_fork_late): the full-grid tcgen05 weight
            # gradient then shares the SMs with the latency-bound mean_bwd_t gather
            # instead of stretching the small dA GEMM it would displace
            late = ws is not None and i != 0 and self.wgrad_fork_late
            if ws is not None and i != 0 and not late:
                fork_wgrad(i, dz)
                forked = True
            elif ws is None or i == 0:
                self._wgrad(i, dz, saved, grads_zeroed)
            if i == 0:
                break
            dA = self._dA(i, dz, saved)
            if late:
                fork_wgrad(i, dz)
                forked = True
            if t_events is not None:
                cs.wait_event(t_events[i])
            dz = self._input_grad(i, dA, saved, transposes)
        if forked:
            cs.wait_stream(ws)

    def _dA(self, i: int, dz, saved) -> torch.Tensor:
        """dA = dz @ W_cat of layer i ([dmean | dh_dst], mpnn.py:82 backward).  Rows
        past the layer's true destination count are zero (dz is zero there; whole
        padding tiles are zero-filled instead of computed)."""
        w = self.wb[i]
        if not self._tc_dA_layer(i):
            return torch.mm(dz, w)
        dA = torch.empty((dz.shape[0], w.shape[1]), dtype=self.act, device=dz.device)
        _lib.check(_lib.lib().sal_tc_gemm_nn(
            dz.data_ptr(), dz.stride(0), dz.shape[0], _lib.ptr(saved[i]["adj"][3]), w.shape[0],
            w.data_ptr(), w.stride(0), w.shape[1], dA.data_ptr(), dA.stride(0), 1,
            _lib.stream_ptr()), "tc_gemm_nn")
        return dA

    def _wgrad(self, i: int, dz, saved, grads_zeroed: bool) -> None:
        L = _lib.lib()
        rec = saved[i]
        a, n_pad = rec["a"], rec["n_pad"]
        if self._tc_wgrad_layer(i):
            gi = self.gp[i]
            # rows past the layer's true destination count carry zero dz
            _lib.check(L.sal_tc_sage_wgrad(dz.data_ptr(), dz.stride(0), a.data_ptr(),
                                           a.stride(0), n_pad, _lib.ptr(rec["adj"][3]),
                                           gi.shape[0], gi.shape[1],
                                           gi.data_ptr(), gi.stride(0),
                                           1 if grads_zeroed else 0, _lib.stream_ptr()),
                       "tc_sage_wgrad")
        else:
            _mm_f32(dz.t(), a[:n_pad], self.gp[i])

    def _input_grad(self, i: int, dA, saved, transposes):
        """dz of layer i-1 from dA = [dmean | dh_dst] of layer i (mean_bwd_t over the
        reverse adjacency, ReLU/dropout backward fused)."""
        L = _lib.lib()
        rec = saved[i]
        a, n_pad = rec["a"], rec["n_pad"]
        f = self.dims[i]
        indptr, src, _, n_dev = rec["adj"]
        rows = a.shape[0]
        cplx = ncplx = None
        if transposes is not None and transposes[i] is not None:
            tindptr, tdst, tw = transposes[i][:3]
            if len(transposes[i]) == 5:   # the workspace's list of source-major rows
                cplx, ncplx = transposes[i][3:]
        else:
            tindptr, tdst, tw = build_transpose(indptr, src, n_dev, n_pad, rows)
        dzp = torch.empty((rows, f), dtype=self.act, device=a.device)
        p = self.p if self.training else 0.0
        mask = saved[i - 1]["mask"]
        m_rows = saved[i - 1]["adj"][3]   # true rows of dz = layer i-1's destinations

        live = i == 1 and self.mbt_live and m_rows is not None and self._tc_wgrad_layer(0)
        if self.mbt_split:
            _lib.check(L.sal_mean_bwd(
                dA.data_ptr(), dA.stride(0), _lib.dtype_code(dA.dtype), f, n_pad,
                _lib.ptr(n_dev), indptr.data_ptr(), src.data_ptr(), tindptr.data_ptr(),
                tdst.data_ptr(), tw.data_ptr(), _lib.ptr(cplx), _lib.ptr(ncplx), rows,
                m_rows.data_ptr() if live else None,
                mask.data_ptr(), p, dzp.data_ptr(), dzp.stride(0), _lib.dtype_code(self.act),
                _lib.stream_ptr()), "mean_bwd")
            return dzp
        if live:
            # dz_0's only reader is layer 0's split-K weight gradient, which reads
            # whole 64-row chunks up to its true row count: skip the padding rows
            _lib.check(L.sal_mean_bwd_t_live(
                dA.data_ptr(), dA.stride(0), _lib.dtype_code(dA.dtype), f, n_pad,
                indptr.data_ptr(), tindptr.data_ptr(), tdst.data_ptr(), tw.data_ptr(), rows,
                m_rows.data_ptr(), mask.data_ptr(), p, dzp.data_ptr(), dzp.stride(0),
                _lib.dtype_code(self.act), _lib.stream_ptr()), "mean_bwd_t_live")
            return dzp
        _lib.check(L.sal_mean_bwd_t(
            dA.data_ptr(), dA.stride(0), _lib.dtype_code(dA.dtype), f, n_pad, indptr.data_ptr(),
            tindptr.data_ptr(), tdst.data_ptr(), tw.data_ptr(), rows, mask.data_ptr(), p,
            dzp.data_ptr(), dzp.stride(0), _lib.dtype_code(self.act), _lib.stream_ptr()),
            "mean_bwd_t")
        return dzp

    # ------------------------------------------------------------- output layer on tcgen05
    def head_ok(self) -> bool:
        """The output layer runs as one tcgen05 kernel (sal_tc_sage_head: logits, loss,
        dlogits, dA and dW; sal_tc_sage_logits_argmax for inference): bf16, 2 f_in =
        128, 256 or 512 (one CTA per 64-wide K block in a cluster), padded classes
        <= 192."""
        k = 2 * self.dims[self.L - 1]
        return (self.tc_head and self.act == torch.bfloat16 and k in (128, 256, 512)
                and self.c_pad <= 192)

    def _head_buffers(self, rows: int, k: int):
        """Persistent dlogits [rows, c_pad] (bf16) and the head kernel's L2 workspace
        (split-K logits partials), sized for `rows` output rows."""
        nbytes = _lib.lib().sal_tc_sage_head_ws_bytes(rows, k, self.c_pad)
        hb = getattr(self, "_hb", None)
        if hb is None or hb[0].shape[0] < rows or hb[1].numel() < nbytes:
            hb = (torch.zeros((rows, self.c_pad), dtype=self.act, device=self.device),
                  torch.empty(nbytes, dtype=torch.uint8, device=self.device))
            self._hb = hb
        return hb[0][:rows], hb[1]

    def loss_backward(self, saved, labels: torch.Tensor, out: torch.Tensor, transposes=None,
                      grads_zeroed: bool = False, loss_zeroed: bool = False,
                      t_events=None) -> torch.Tensor:
        """After forward(..., head=True): the output layer (logits in TMEM only, the loss
        *out += mean NLL, dlogits, its dA and dW) in one tcgen05 kernel, then the
        backward of the layers below.  grads_zeroed: the caller zeroed the tcgen05
        weight-gradient blocks (the output layer's included)."""
        L = _lib.lib()
        i = self.L - 1
        rec = saved[i]
        a, n_pad = rec["a"], rec["n_pad"]
        if not loss_zeroed:
            out.zero_()
        gi = self.gp[i]
        if not grads_zeroed:
            gi.zero_()
        w = self.wb[i]
        dA = torch.empty((n_pad, a.shape[1]), dtype=self.act, device=a.device)
        dlog, ws = self._head_buffers(n_pad, a.shape[1])
        _lib.check(L.sal_tc_sage_head(
            a.data_ptr(), a.stride(0), n_pad, _lib.ptr(rec["adj"][3]), a.shape[1], w.data_ptr(),
            w.stride(0), self.c_pad, self.dims[-1], labels.data_ptr(), labels.numel(),
            out.data_ptr(), dlog.data_ptr(), dlog.stride(0), dA.data_ptr(), dA.stride(0),
            gi.data_ptr(), gi.stride(0), ws.data_ptr(), ws.numel(), _lib.stream_ptr()),
            "tc_sage_head")
        if i == 0:
            return out
        if t_events is not None:
            torch.cuda.current_stream().wait_event(t_events[i])
        dz = self._input_grad(i, dA, saved, transposes)
        self._backward_below(i - 1, dz, saved, transposes, grads_zeroed, t_events)
        return out

    def score(self, saved, labels: torch.Tensor, counts: torch.Tensor) -> None:
        """After forward(..., head=True) in eval mode: counts[0] += correct argmax
        predictions, counts[1] += labelled rows (logits never leave TMEM)."""
        i = self.L - 1
        rec = saved[i]
        a, n_pad = rec["a"], rec["n_pad"]
        w = self.wb[i]
        _, ws = self._head_buffers(n_pad, a.shape[1])
        _lib.check(_lib.lib().sal_tc_sage_logits_argmax(
            a.data_ptr(), a.stride(0), n_pad, _lib.ptr(rec["adj"][3]), a.shape[1], w.data_ptr(),
            w.stride(0), self.c_pad, self.dims[-1], labels.data_ptr(), labels.numel(),
            counts.data_ptr(), ws.data_ptr(), ws.numel(), _lib.stream_ptr()),
            "tc_sage_logits_argmax")

    @torch.no_grad()
    def predict(self, x, adjs, x_global=None, cat: bool = False):
        was = self.training
        self.training = False
        try:
            a0 = x if cat else self.cat_input(x)
            logits, _ = self.forward(a0, adjs, x_global)
        finally:
            self.training = was
        return logits


def build_transpose(indptr, src, n_dst_dev, n_pad: int, n_src_rows: int, out=None, ws=None,
                    ws_zeroed: bool = False):
    """Reverse adjacency (tindptr [n_src_rows+1], tdst, tw [edges]) of one MFG layer."""
    L = _lib.lib()
    dev = indptr.device
    if out is None:
        tindptr = torch.empty(n_src_rows + 1, dtype=torch.int32, device=dev)
        tdst = torch.empty(max(src.numel(), 1), dtype=torch.int32, device=dev)
        tw = torch.empty(max(src.numel(), 1), dtype=torch.float32, device=dev)
    else:
        tindptr, tdst, tw = out[:3]
    if ws is None:
        ws = torch.empty(L.sal_transpose_ws_bytes(n_src_rows), dtype=torch.uint8, device=dev)
    _lib.check(L.sal_transpose_build(indptr.data_ptr(), src.data_ptr(), _lib.ptr(n_dst_dev),
                                     n_pad, n_src_rows, src.numel(), tindptr.data_ptr(),
                                     tdst.data_ptr(), tw.data_ptr(), ws.data_ptr(),
                                     1 if ws_zeroed else 0, _lib.stream_ptr()),
               "transpose_build")
    return tindptr, tdst, tw


def _mm_f32(a: torch.Tensor, b: torch.Tensor, out: torch.Tensor) -> None:
    """out (fp32) = a @ b; 16-bit operands accumulate and store in fp32 (cuBLAS)."""
    if a.dtype == torch.float32:
        torch.mm(a, b, out=out)
    else:
        torch.mm(a, b, out_dtype=torch.float32, out=out)
