"""The drop-in MFG build (sal_sample_mfg, full 3-hop MFG with relabel) alone on
papers-shape batches: K batches captured in one CUDA graph and replayed R times
(median per batch), then the same K batches on 8 streams at once.  For A/B of
library builds: SAL_LIB=<variant .so> python tools/mfg_ab.py [K] [R]
"""
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2110_08450_b200 import make_epoch_plan  # noqa: E402
from paper_2110_08450_b200.sampler import FanoutSpec, MfgWorkspace  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 32
R = int(sys.argv[2]) if len(sys.argv) > 2 else 7
dg, train, _, _ = bench.build_data("papers")
plan = make_epoch_plan(train, 1024, 1)
fan = FanoutSpec((15, 10, 5))
seeds = torch.zeros(len(train), dtype=torch.int64, device="cuda")
perm = np.concatenate([b.dst_ids for b in plan.batches])
seeds[:len(perm)].copy_(torch.from_numpy(perm))
descs = [torch.tensor([plan.batches[b].batch_id, b * 1024, len(plan.batches[b])],
                      dtype=torch.int64, device="cuda") for b in range(K)]
ws = MfgWorkspace(dg.num_nodes, fan, 1024, device="cuda")
side = torch.cuda.Stream()
with torch.cuda.stream(side):
    for b in range(2):
        ws.run(dg, seeds, descs[b], 1, 0, side)
torch.cuda.synchronize()
digest = ws.read_extents()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    for b in range(K):
        ws.run(dg, seeds, descs[b], 1, 0, torch.cuda.current_stream())
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ts = []
for _ in range(R):
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) * 1e3 / K)
# 8 concurrent streams, each its own workspace and graph of K/8 batches
P = 8
wss = [MfgWorkspace(dg.num_nodes, fan, 1024, device="cuda") for _ in range(P)]
sts = [torch.cuda.Stream() for _ in range(P)]
gs = []
for p in range(P):
    with torch.cuda.stream(sts[p]):
        wss[p].run(dg, seeds, descs[p], 1, 0, sts[p])
    torch.cuda.synchronize()
    gp = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gp, stream=sts[p]):
        for b in range(p, K, P):
            wss[p].run(dg, seeds, descs[b], 1, 0, sts[p])
    gs.append(gp)
torch.cuda.synchronize()
tp = []
for _ in range(R):
    torch.cuda.synchronize()
    e0.record()
    for p in range(P):
        sts[p].wait_event(e0)
        with torch.cuda.stream(sts[p]):
            gs[p].replay()
    for p in range(P):
        torch.cuda.current_stream().wait_stream(sts[p])
    e1.record()
    torch.cuda.synchronize()
    tp.append(e0.elapsed_time(e1) * 1e3 / K)
print(f"lib={os.environ.get('SAL_LIB', 'default')} K={K} graph us/batch median "
      f"{np.median(ts):.1f} (min {min(ts):.1f}); 8 streams us/batch median {np.median(tp):.1f} "
      f"(min {min(tp):.1f}); extents of batch 1 {digest}")
