"""cuBLAS timings for the GraphSAGE step's GEMM shapes (papers shape, padded).

Compares the weight-gradient GEMM layouts / output dtypes so the fused model
can pick the fastest formulation.  Run under gpurun: python tools/gemm_shapes.py
"""
import torch

dev = "cuda"
bf = torch.bfloat16


def t(fn, it=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(it):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / it * 1e3


for name, n, k, fo in [("L0", 67584, 256, 256), ("L1", 6144, 512, 256), ("L2", 1024, 512, 172)]:
    A = torch.randn(n, k, device=dev, dtype=bf)        # cat activations [n, 2f]
    W = torch.randn(fo, k, device=dev, dtype=bf)       # [f_out, 2f]
    WT = W.t().contiguous()                            # [2f, f_out]
    dz = torch.randn(n, fo, device=dev, dtype=bf)
    g32 = torch.empty(fo, k, device=dev)
    g32t = torch.empty(k, fo, device=dev)
    g16 = torch.empty(fo, k, device=dev, dtype=bf)
    print(f"== {name}: n={n} K={k} f_out={fo}")
    print(f"  fwd  A@W^T (W row-major)           {t(lambda: torch.mm(A, W.t())):7.1f} us")
    print(f"  fwd  A@WT  (W stored transposed)   {t(lambda: torch.mm(A, WT)):7.1f} us")
    print(f"  dW   dz^T@A -> fp32               {t(lambda: torch.mm(dz.t(), A, out_dtype=torch.float32, out=g32)):7.1f} us")
    print(f"  dWT  A^T@dz -> fp32               {t(lambda: torch.mm(A.t(), dz, out_dtype=torch.float32, out=g32t)):7.1f} us")
    print(f"  dW   dz^T@A -> bf16               {t(lambda: torch.mm(dz.t(), A, out=g16)):7.1f} us")
    print(f"  dA   dz@W                         {t(lambda: torch.mm(dz, W)):7.1f} us")
    print(f"  dA   dz@WT^T                      {t(lambda: torch.mm(dz, WT.t())):7.1f} us")
