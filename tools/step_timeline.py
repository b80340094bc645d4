"""Kernel timeline of a few overlapped training steps (CUPTI via torch.profiler):
start offset, duration, stream, name — shows which chain is critical and where
the gaps are.

python tools/step_timeline.py [steps] [--no-prep]   (under gpurun; --no-prep replays the
step with the batch preparation removed: the training chain alone, stale inputs)
"""
import sys
from pathlib import Path

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2110_08450_b200.train import TrainConfig, Trainer  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
steps = int(args[0]) if args else 3
dg, train, _, _ = bench.build_data("papers")
tr = Trainer(dg, train, TrainConfig(gather_free=True))
tr.set_epoch(0)
tr.begin_epoch(False)
tr.run_steps(0, 12)
torch.cuda.synchronize()
if "--no-prep" in sys.argv:
    from paper_2110_08450_b200 import sampler
    sampler.MfgWorkspace.run = lambda self, *a, **k: None
    sampler.MfgWorkspace.aggregate = lambda self, *a, **k: None
    tr.graphs.clear()
    tr.run_steps(12, 4)
    torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    tr.run_steps(12, steps)
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
