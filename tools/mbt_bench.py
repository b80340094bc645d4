"""Time sal_mean_bwd_t (the input gradient of layer 1: dz_0 for the layer-0
destination rows) alone on the papers-shape layer: 6144 destinations x 10
sampled edges over 67584 source rows, f = 256, bf16, p = 0.5.

python tools/mbt_bench.py [--split]   (under gpurun)
"""
import ctypes
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2110_08450_b200 import _lib  # noqa: E402
from paper_2110_08450_b200.model import build_transpose  # noqa: E402

L = _lib.lib()
dev = "cuda"
torch.manual_seed(0)
n_dst, fan, rows, f = 6144, 10, 67584, 256
rng = np.random.default_rng(0)
indptr = torch.from_numpy(np.arange(0, (n_dst + 1) * fan, fan, dtype=np.int32)).to(dev)
# sampled sources: mostly distinct new nodes past the destinations, as after the relabel
src_np = rng.permutation(np.arange(n_dst, rows))[:n_dst * fan].astype(np.int32)
src_np[::7] = rng.integers(0, rows, size=src_np[::7].shape[0])
src = torch.from_numpy(src_np).to(dev)
n_dev = torch.tensor([n_dst], dtype=torch.int64, device=dev)
tws = torch.zeros(L.sal_transpose_ws_bytes(rows), dtype=torch.uint8, device=dev)
tind, tdst, tw = build_transpose(indptr, src, n_dev, n_dst, rows, ws=tws, ws_zeroed=True)
_lo, _co = ctypes.c_int64(), ctypes.c_int64()
L.sal_transpose_complex_list(rows, ctypes.byref(_lo), ctypes.byref(_co))
cplx = tws[_lo.value:_lo.value + 4 * rows].view(torch.int32)
ncplx = tws[_co.value:_co.value + 4].view(torch.int32)
dA = (torch.randn(n_dst, 2 * f, device=dev) * 0.1).to(torch.bfloat16)
mask = torch.from_numpy(rng.integers(0, 256, size=rows * f // 8, dtype=np.uint8)).to(dev)
dz = torch.empty(rows, f, device=dev, dtype=torch.bfloat16)


SPLIT = "--split" in sys.argv


def run():
    if SPLIT:
        _lib.check(L.sal_mean_bwd(dA.data_ptr(), dA.stride(0), _lib.SAL_BF16, f, n_dst,
                                  n_dev.data_ptr(), indptr.data_ptr(), src.data_ptr(),
                                  tind.data_ptr(), tdst.data_ptr(), tw.data_ptr(),
                                  cplx.data_ptr(), ncplx.data_ptr(), rows, None,
                                  mask.data_ptr(), 0.5, dz.data_ptr(), dz.stride(0),
                                  _lib.SAL_BF16, _lib.stream_ptr()), "mean_bwd")
        return
    _lib.check(L.sal_mean_bwd_t(dA.data_ptr(), dA.stride(0), _lib.SAL_BF16, f, n_dst,
                                indptr.data_ptr(), tind.data_ptr(), tdst.data_ptr(),
                                tw.data_ptr(), rows, mask.data_ptr(), 0.5, dz.data_ptr(),
                                dz.stride(0), _lib.SAL_BF16, _lib.stream_ptr()), "mbt")


flush = torch.ones(32 << 20, dtype=torch.int64, device=dev)
for _ in range(3):
    run()
torch.cuda.synchronize()
ts = []
for _ in range(20):
    flush.sum()      # L2 holds clean unrelated lines (a read flush: no write-back behind us)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    run()
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b) * 1e3)
byts = rows * f * 2 + rows * f // 8 + n_dst * fan * (2 * f + 12) + (rows + 1) * 4
t = float(np.median(ts))
print(f"{'mean_bwd(split)' if SPLIT else 'mean_bwd_t'}  rows {rows}  edges {n_dst * fan}  {t:.1f} us  {byts / t / 1e3:.0f} GB/s "
      f"(algorithmic {byts / 1e6:.1f} MB)")
# checksum for A/B of kernel variants
bits = dz.view(torch.int16).to(torch.int64)
w = torch.arange(1, bits.shape[1] + 1, device=dev, dtype=torch.int64)
print("checksum", int(((bits * w).sum(1) * torch.arange(1, rows + 1, device=dev)).sum()))
