"""A/B the training step on the papers shape: one data build, several TrainConfig
variants, each timed over a full epoch twice (interleaved) with CUDA events.

python tools/step_ab.py [--steps N] [variant ...]   (under gpurun)
variant = name:key=val,key=val   e.g.  notc:sampler_tcount=0  nofirst:first_edge=0
"""
import argparse
import ast
import gc
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2110_08450_b200.sampler import FanoutSpec  # noqa: E402
from paper_2110_08450_b200.train import TrainConfig, Trainer  # noqa: E402


def parse_variant(s):
    """name:key=val,...; a key `m.attr` sets FusedSAGE.attr (a Python literal; use
    `;` for commas inside it, e.g. m.tc_fwd_k=(256;)) after the trainer is built."""
    name, _, kv = s.partition(":")
    out = {}
    for item in filter(None, kv.split(",")):
        k, v = item.split("=")
        if k.startswith("m."):
            out[k] = ast.literal_eval(v.replace(";", ","))
            continue
        f = TrainConfig.__dataclass_fields__[k]
        out[k] = (v not in ("0", "false")) if f.type in (bool, "bool") else type(f.default)(v)
    return name, out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=0)
    ap.add_argument("--shape", default="papers")
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--fanouts", default="15,10,5")
    ap.add_argument("variants", nargs="*")
    a = ap.parse_args()
    variants = [("base", {})] + [parse_variant(v) for v in a.variants]
    dg, train, _, _ = bench.build_data(a.shape)
    res = {n: [] for n, _ in variants}
    for rep in range(a.reps):
        for name, kw in variants:
            tr = Trainer(dg, train, TrainConfig(gather_free=True, fanouts=FanoutSpec.parse(a.fanouts),
                                                **{k: v for k, v in kw.items()
                                                   if not k.startswith("m.")}))
            for k, v in kw.items():
                if k.startswith("m."):
                    setattr(tr.model, k[2:], v)
            spe = tr.set_epoch(0)
            n = a.steps or spe
            tr.begin_epoch(False)
            tr.run_steps(0, min(8, spe))
            torch.cuda.synchronize()
            tr.set_epoch(1)
            tr.begin_epoch(False)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            tr.run_steps(0, min(n, spe))
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / min(n, spe)
            res[name].append(ms)
            print(f"rep {rep} {name:12s} {ms * 1e3:8.1f} us/step  loss {tr.last_loss.item():.3f}",
                  flush=True)
            del tr
            gc.collect()
            torch.cuda.empty_cache()
    for name, v in res.items():
        print(f"{name:12s} min {min(v) * 1e3:8.1f} us/step  all {[round(x * 1e3, 1) for x in v]}")


if __name__ == "__main__":
    main()
