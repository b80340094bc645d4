"""Time the layer-0 tcgen05 kernels against cuBLAS on the papers-shape sizes.

python tools/tc_bench.py   (under gpurun)
"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2110_08450_b200 import _lib  # noqa: E402

L = _lib.lib()
M = 67584
dev = "cuda"
A = (torch.randn(M, 512, device=dev) * 0.5).to(torch.bfloat16)[:, :256]
W = (torch.randn(256, 256, device=dev) * 0.06).to(torch.bfloat16)
Y = torch.zeros(M, 512, device=dev, dtype=torch.bfloat16)[:, 256:]
mask = torch.zeros(M * 32, dtype=torch.uint8, device=dev)
dz = (torch.randn(M, 256, device=dev) * 0.1).to(torch.bfloat16)
dW = torch.zeros(256, 256, device=dev)
salt = torch.zeros(1, dtype=torch.int64, device=dev)
st = lambda: _lib.stream_ptr()  # noqa: E731


def t(fn, it=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(it):
            fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g.replay()
    torch.cuda.synchronize()
    a.record()
    g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / it * 1e3


def fwd_tma():
    _lib.check(L.sal_tc_sage_fwd(A.data_ptr(), A.stride(0), M, None, W.data_ptr(), 256, 256,
                                 Y.data_ptr(), Y.stride(0), mask.data_ptr(), 0.5, 1,
                                 salt.data_ptr(), 1, st()))


def fwd_tma_plain():   # no ReLU/dropout: the epilogue only converts (isolates its cost)
    _lib.check(L.sal_tc_sage_fwd(A.data_ptr(), A.stride(0), M, None, W.data_ptr(), 256, 256,
                                 Y.data_ptr(), Y.stride(0), mask.data_ptr(), 0.0, 1,
                                 salt.data_ptr(), 0, st()))


def fwd_simple():
    _lib.check(L.sal_tc_sage_fwd_simple(A.data_ptr(), A.stride(0), M, W.data_ptr(), 256, 256,
                                        Y.data_ptr(), Y.stride(0), mask.data_ptr(), 0.5, 1,
                                        salt.data_ptr(), 1, st()))


def fwd_cublas():
    z = torch.mm(A, W.t())
    _lib.check(L.sal_relu_dropout_fwd(z.data_ptr(), z.stride(0), Y.data_ptr(), Y.stride(0), M,
                                      256, _lib.SAL_BF16, mask.data_ptr(), 0.5, 1,
                                      salt.data_ptr(), st()))


def wg_tma():
    _lib.check(L.sal_tc_sage_wgrad(dz.data_ptr(), dz.stride(0), A.data_ptr(), A.stride(0), M,
                                   None, 256, 256, dW.data_ptr(), dW.stride(0), 0, st()))


def wg_simple():
    _lib.check(L.sal_tc_sage_wgrad_simple(dz.data_ptr(), dz.stride(0), A.data_ptr(),
                                          A.stride(0), M, 256, 256, dW.data_ptr(),
                                          dW.stride(0), st()))


def wg_cublas():
    torch.mm(dz.t(), A, out_dtype=torch.float32, out=dW)


bytes_fwd = M * 256 * 2 * 2 + M * 32
bytes_wg = M * 256 * 2 * 2
for name, fn, nb in [("fwd tma (gemm+relu/dropout)", fwd_tma, bytes_fwd),
                     ("fwd tma (gemm only)", fwd_tma_plain, bytes_fwd),
                     ("fwd simple", fwd_simple, bytes_fwd),
                     ("fwd cublas + relu_dropout", fwd_cublas, bytes_fwd),
                     ("wgrad tma", wg_tma, bytes_wg), ("wgrad simple", wg_simple, bytes_wg),
                     ("wgrad cublas fp32 out", wg_cublas, bytes_wg)]:
    us = t(fn)
    print(f"{name:32s} {us:7.1f} us  {nb / us / 1e3:7.0f} GB/s")
