"""f3: GPU design-space sweep on a TRCE hop replay (reference bench.py methodology).

Builds the bench graph (device-generated, `--shape`), records a trace of the
first B batches of the epoch plan, sweeps sweep.default_grid() (lanes per
destination x sampler grid cap x id-table load) with digest guarding, and
writes the CSV plus a per-hop summary.

python tools/sweep.py [--shape papers] [--batches 16] [--reps 5] [--out gpurun_out/sweep]
"""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2110_08450_b200 import FanoutSpec, make_epoch_plan  # noqa: E402
from paper_2110_08450_b200 import harness as S  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="papers")
    ap.add_argument("--batches", type=int, default=16)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--fanouts", default="15,10,5")
    ap.add_argument("--out", default="gpurun_out/sweep")
    a = ap.parse_args()
    out = Path(a.out)
    out.mkdir(parents=True, exist_ok=True)
    dg, train, _, _ = bench.build_data(a.shape)
    fan = FanoutSpec(tuple(int(x) for x in a.fanouts.split(",")))
    plan = make_epoch_plan(train, 1024, 1)

    class P:
        batches = plan.batches[:a.batches]
    t0 = time.perf_counter()
    tr = S.record_trace(dg, P(), fan, 1, path=out / "trace.trce")
    rec_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    res = S.sweep(tr, dg, S.default_grid(), S.DeviceVariant(), path=out / "sweep.csv",
                  repetitions=a.reps)
    sweep_s = time.perf_counter() - t0
    edges = {}
    for r in tr.records:
        edges[r.hop] = edges.get(r.hop, 0) + len(r.dst_ids)
    summary = {"shape": a.shape, "batches": a.batches, "records": len(tr.records),
               "record_s": round(rec_s, 2), "sweep_s": round(sweep_s, 2),
               "baseline": res.baseline, "dst_per_hop": edges, "best": {}}
    for hop in sorted({h for _, h, _, _ in res.rows}):
        rows = sorted((t, v) for v, h, t, _ in res.rows if h == hop)
        base = next(t for v, h, t, _ in res.rows if h == hop and v == res.baseline)
        summary["best"][hop] = {"variant": rows[0][1], "us_per_batch": round(1e6 * rows[0][0] / a.batches, 2),
                                "baseline_us_per_batch": round(1e6 * base / a.batches, 2),
                                "worst": rows[-1][1],
                                "worst_us_per_batch": round(1e6 * rows[-1][0] / a.batches, 2)}
    (out / "summary.json").write_text(json.dumps(summary, indent=1))
    print(json.dumps(summary))


if __name__ == "__main__":
    main()
