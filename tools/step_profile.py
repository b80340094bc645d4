"""Per-kernel time of the papers-shape training step, warm caches, real clocks.

CUPTI kernel records (torch.profiler) over N graph-replayed steps; the prep and
compute streams overlap as in bench.py, so per-kernel times include sharing.
With --serial the prep of step i+1 runs on the compute stream (no overlap).

python tools/step_profile.py [--steps 50] [--serial]   (under gpurun)
"""
import argparse
import sys
from collections import defaultdict
from pathlib import Path

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2110_08450_b200.train import TrainConfig, Trainer  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--shape", default="papers")
    ap.add_argument("--serial", action="store_true")
    a = ap.parse_args()
    dg, train, _, _ = bench.build_data(a.shape)
    tr = Trainer(dg, train, TrainConfig(gather_free=True))
    if a.serial:
        tr.prep_stream = None
    tr.set_epoch(0)
    tr.begin_epoch(False)
    tr.run_steps(0, 8)
    torch.cuda.synchronize()
    tr.set_epoch(1)
    tr.begin_epoch(False)
    tr.run_steps(0, 4)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        tr.run_steps(4, a.steps)
        torch.cuda.synchronize()
    agg = defaultdict(lambda: [0, 0.0])
    t0, t1 = None, None
    for ev in prof.events():
        if ev.device_type.name != "CUDA":
            continue
        name = ev.name.split("(")[0].replace("void ", "")[:80]
        agg[name][0] += 1
        agg[name][1] += ev.device_time_total
        s, e = ev.time_range.start, ev.time_range.end
        t0 = s if t0 is None else min(t0, s)
        t1 = e if t1 is None else max(t1, e)
    tot = sum(v[1] for v in agg.values())
    print(f"{'us/step':>9} {'calls/step':>10}  kernel")
    for name, (c, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{us / a.steps:9.1f} {c / a.steps:10.1f}  {name}")
    print(f"sum of kernel time {tot / a.steps:.1f} us/step; wall span {(t1 - t0) / a.steps:.1f} "
          f"us/step over {a.steps} steps ({'serial' if a.serial else 'overlapped'})")


if __name__ == "__main__":
    main()
