"""Fused last hop (sal_sample_aggregate) alone on papers-shape batches, against the
unfused chain it replaces (edges-only last hop -> layer-0 mean -> self-row gather).

python tools/fused_bench.py [batches]   (under gpurun; SAL_SAMPLE_MEAN_BPS=1|2|3 picks the
resident blocks per SM of the fused kernel)
"""
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2110_08450_b200 import _lib, make_epoch_plan  # noqa: E402
from paper_2110_08450_b200.prep import gather_rows  # noqa: E402
from paper_2110_08450_b200.sampler import FanoutSpec, MfgWorkspace  # noqa: E402

nb = int(sys.argv[1]) if len(sys.argv) > 1 else 20
dg, train, _, _ = bench.build_data("papers")
plan = make_epoch_plan(train, 1024, 1)
fan = FanoutSpec((15, 10, 5))
x = dg.features
f = x.shape[1]
ws = MfgWorkspace(dg.num_nodes, fan, 1024, device="cuda", last_hop_edges=True)
fws = MfgWorkspace(dg.num_nodes, fan, 1024, device="cuda", last_hop_fused=True)
h = ws.num_hops - 1
out_a = torch.zeros((ws.node_cap[h], 2 * f), dtype=torch.bfloat16, device="cuda")
out_b = torch.zeros_like(out_a)
seeds = torch.zeros(len(train), dtype=torch.int64, device="cuda")
perm = np.concatenate([b.dst_ids for b in plan.batches])
seeds[:len(perm)].copy_(torch.from_numpy(perm))
L = _lib.lib()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(7)]
st = torch.cuda.current_stream()
tot = np.zeros(5)
equal = 0
for b in range(nb + 1):
    desc = torch.tensor([plan.batches[b].batch_id, b * 1024, len(plan.batches[b])],
                        dtype=torch.int64, device="cuda")
    ev[0].record(st)
    ws.run(dg, seeds, desc, 1, 0)
    ev[1].record(st)
    _lib.check(L.sal_segment_mean_fwd_ex(
        ws.dst_indptr[h].data_ptr(), ws.src_glob.data_ptr(), ws.sizes[h:h + 1].data_ptr(),
        ws.node_cap[h], x.data_ptr(), _lib.SAL_F16, x.stride(0), f, out_a.data_ptr(),
        _lib.SAL_BF16, out_a.stride(0), _lib.SAL_SEG_NO_PAD_FILL, _lib.stream_ptr()), "mean")
    ev[2].record(st)
    gather_rows(x, ws.globals, out_a[:, f:], n=ws.node_cap[h], n_dev=ws.sizes[h:h + 1])
    ev[3].record(st)
    fws.run(dg, seeds, desc, 1, 0)
    ev[4].record(st)
    fws.aggregate(dg, x, out_b, f, desc, 1, 0)
    ev[5].record(st)
    torch.cuda.synchronize()
    n = int(ws.sizes[h].item())
    equal += int(torch.equal(out_a[:n].view(torch.int16), out_b[:n].view(torch.int16)))
    if b:
        tot += [ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2]), ev[2].elapsed_time(ev[3]),
                ev[3].elapsed_time(ev[4]), ev[4].elapsed_time(ev[5])]
tot *= 1e3 / nb
print(f"bps={os.environ.get('SAL_SAMPLE_MEAN_BPS', 'default')} batches={nb} equal={equal}/{nb + 1}")
print(f"  unfused: mfg(3 hops) {tot[0]:.1f} us + l0 mean {tot[1]:.1f} us + self gather "
      f"{tot[2]:.1f} us = {tot[0] + tot[1] + tot[2]:.1f} us")
print(f"  fused:   mfg(2 hops) {tot[3]:.1f} us + sample_mean {tot[4]:.1f} us = "
      f"{tot[3] + tot[4]:.1f} us")
