"""Kernel timeline of a few sampled-inference steps (Evaluator, (20,20,20)) at
papers shape (CUPTI via torch.profiler).

python tools/infer_timeline.py [steps]   (under gpurun)
"""
import sys
from pathlib import Path

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2110_08450_b200 import FanoutSpec  # noqa: E402
from paper_2110_08450_b200.train import Evaluator, TrainConfig, Trainer  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
dg, train, test, _ = bench.build_data("papers")
tr = Trainer(dg, train, TrainConfig(gather_free=True))
ev = Evaluator(dg, tr.model, FanoutSpec((20, 20, 20)), 1024, 8)
n = ev.set_ids(test)
for p in range(2):
    ev._capture(p)
ev.begin()
ev.steps(0, 10)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    ev.steps(10, steps)
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
evs.sort(key=lambda e: e.time_range.start)
t0 = evs[0].time_range.start
streams = {}
for e in evs:
    sid = streams.setdefault(getattr(e, "device_resource_id", 0), len(streams))
    name = e.name.split("(")[0].replace("void ", "").replace("sal::", "")[:60]
    print(f"{e.time_range.start - t0:8.1f} {e.time_range.end - t0:8.1f} "
          f"{e.time_range.end - e.time_range.start:7.1f}  s{sid}  {name}")
