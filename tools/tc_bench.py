"""Time the tcgen05 kernels of the step against cuBLAS on the papers-shape sizes.

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


def fwd_cublas():
    z = torch.mm(A, W.t())
    _lib.check(L.sal_relu_dropout_fwd(z.data_ptr(), z.stride(0), Y.data_ptr(), Y.stride(0), M,
                                      256, _lib.SAL_BF16, mask.data_ptr(), 0.5, 1,
                                      salt.data_ptr(), st()))


def wg_tma():
    _lib.check(L.sal_tc_sage_wgrad(dz.data_ptr(), dz.stride(0), A.data_ptr(), A.stride(0), M,
                                   None, 256, 256, dW.data_ptr(), dW.stride(0), 0, st()))


def wg_cublas():
    torch.mm(dz.t(), A, out_dtype=torch.float32, out=dW)


# the rest of the step: output layer (1024 x 512 -> 176 classes), its dA and dW,
# the hidden layer's dA (6144 x 256 -> 512)
B2, C2, CP = 1024, 172, 176
A2 = (torch.randn(B2, 512, device=dev) * 0.5).to(torch.bfloat16)
W2 = (torch.randn(CP, 512, device=dev) * 0.05).to(torch.bfloat16)
lab = torch.randint(0, C2, (B2,), device=dev)
loss = torch.zeros((), device=dev)
dlog = torch.zeros(B2, CP, device=dev, dtype=torch.bfloat16)
dA2 = torch.zeros(B2, 512, device=dev, dtype=torch.bfloat16)
dW2 = torch.zeros(CP, 512, device=dev)
M1 = 6144
dz1 = (torch.randn(M1, 256, device=dev) * 0.1).to(torch.bfloat16)
W1 = (torch.randn(256, 512, device=dev) * 0.05).to(torch.bfloat16)
dA1 = torch.zeros(M1, 512, device=dev, dtype=torch.bfloat16)


hws = torch.empty(L.sal_tc_sage_head_ws_bytes(B2, 512, CP), dtype=torch.uint8, device=dev)


def head_tc():   # logits + loss + dlogits + dA + dW in one kernel
    _lib.check(L.sal_tc_sage_head(A2.data_ptr(), 512, B2, None, 512, W2.data_ptr(), 512, CP, C2,
                                  lab.data_ptr(), B2, loss.data_ptr(), dlog.data_ptr(), CP,
                                  dA2.data_ptr(), 512, dW2.data_ptr(), 512, hws.data_ptr(),
                                  hws.numel(), st()))


def head_cublas():   # the same four results the unfused way
    logits_nll_cublas()
    dA2_cublas()
    dW2_cublas()


def logits_nll_cublas():
    z = torch.mm(A2, W2.t())
    _lib.check(L.sal_lsm_nll(z.data_ptr(), z.stride(0), B2, C2, _lib.SAL_BF16, lab.data_ptr(),
                             loss.data_ptr(), dlog.data_ptr(), CP, st()))


def dA2_cublas():
    torch.mm(dlog, W2, out=dA2)


def dW2_cublas():
    torch.mm(dlog.t(), A2, out_dtype=torch.float32, out=dW2)


def dA1_tc():
    _lib.check(L.sal_tc_gemm_nn(dz1.data_ptr(), 256, M1, None, 256, W1.data_ptr(), 512, 512,
                                dA1.data_ptr(), 512, 1, st()))


def dA1_cublas():
    torch.mm(dz1, W1, out=dA1)


bytes_fwd = M * 256 * 2 * 2 + M * 32
bytes_wg = M * 256 * 2 * 2
CASES = [("fwd tma (gemm+relu/dropout)", fwd_tma, bytes_fwd),
                     ("fwd tma (gemm only)", fwd_tma_plain, bytes_fwd),
                     ("fwd cublas + relu_dropout", fwd_cublas, bytes_fwd),
                     ("wgrad tma", wg_tma, bytes_wg),
                     ("wgrad cublas fp32 out", wg_cublas, bytes_wg),
                     ("out layer fused tc", head_tc, B2 * 512 * 2 * 2),
                     ("out layer cublas x3 + lsm_nll", head_cublas, B2 * 512 * 2 * 2),
                     ("out logits cublas + lsm_nll", logits_nll_cublas, B2 * 512 * 2 + B2 * CP * 2),
                     ("out dA cublas", dA2_cublas, B2 * CP * 2 + B2 * 512 * 2),
                     ("out dW cublas", dW2_cublas, B2 * CP * 2 + B2 * 512 * 2),
                     ("hidden dA tc", dA1_tc, M1 * 256 * 2 + M1 * 512 * 2),
                     ("hidden dA cublas", dA1_cublas, M1 * 256 * 2 + M1 * 512 * 2)]

if __name__ == "__main__":
    for name, fn, nb in CASES:
        us = t(fn)
        print(f"{name:32s} {us:7.1f} us  {nb / us / 1e3:7.0f} GB/s")
