"""run_epoch_prep (the drop-in batch-preparation path, reference contract: full MFG,
f32 features, labels) at P = 1, 2, 4, 8 concurrent batches on the papers shape, with
the host time split into launch / wait / finish per batch.

python tools/prep_scaling.py [batches] [P,P,...]   (under gpurun)
"""
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2110_08450_b200.prep as P  # noqa: E402
from paper_2110_08450_b200 import FanoutSpec, PrepConfig, make_epoch_plan, run_epoch_prep  # noqa: E402

nb = int(sys.argv[1]) if len(sys.argv) > 1 else 160
dg, train, _, _ = bench.build_data("papers")
plan = make_epoch_plan(train, 1024, 1)
sub = P.EpochPlan(batches=plan.batches[:nb], batch_size=1024, shuffle_seed=0)
x = dg.feature_view()
acc = {"launch": 0.0, "finish": 0.0}
orig_prep, orig_finish = P._prep_one, P._finish_slot


def prep_one(*a, **k):
    t = time.perf_counter()
    orig_prep(*a, **k)
    acc["launch"] += time.perf_counter() - t


def finish(*a, **k):
    t = time.perf_counter()
    r = orig_finish(*a, **k)
    acc["finish"] += time.perf_counter() - t
    return r


P._prep_one, P._finish_slot = prep_one, finish
ps = [int(v) for v in sys.argv[2].split(",")] if len(sys.argv) > 2 else [1, 2, 4, 8]
for p in ps:
    for delivery in ("in_order", "completion_order"):
        cfg = PrepConfig(num_workers=p, fanouts=FanoutSpec((15, 10, 5)), delivery=delivery,
                         feature_dtype="f32")
        for _ in run_epoch_prep(dg, x, dg.labels, P.EpochPlan(batches=plan.batches[:2 * p],
                                                              batch_size=1024, shuffle_seed=0),
                                cfg, 1):
            pass
        torch.cuda.synchronize()
        acc["launch"] = acc["finish"] = 0.0
        t0 = time.perf_counter()
        for b in run_epoch_prep(dg, x, dg.labels, sub, cfg, 1):
            pass
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        print(f"P={p} {delivery:16s} {wall / nb * 1e6:7.1f} us/batch  epoch {wall * len(plan) / nb:.3f} s"
              f"  host launch {acc['launch'] / nb * 1e6:6.1f} us  finish(wait+build) "
              f"{acc['finish'] / nb * 1e6:6.1f} us", flush=True)
