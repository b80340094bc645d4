"""What-if bounds: the step with one piece removed (wrong results; timing only)."""
import sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench
from paper_2110_08450_b200.train import TrainConfig, Trainer
from paper_2110_08450_b200 import sampler, model

dg, train, _, _ = bench.build_data("papers")
orig = {}
def patch(cls, name, fn):
    orig[(cls, name)] = getattr(cls, name)
    setattr(cls, name, fn)
def unpatch():
    for (cls, name), f in orig.items():
        setattr(cls, name, f)
    orig.clear()

def ig(self, i, dA, saved, transposes):
    rec = saved[i]
    return torch.empty((rec["a"].shape[0], self.dims[i]), dtype=self.act, device=dA.device)

def no_agg(self, *a, **k):
    self.reset_tables()   # called on the stream aggregate() would have run on


modes = {
    "base": lambda: None,
    "no_hops": lambda: patch(sampler.MfgWorkspace, "run", lambda self, *a, **k: None),
    # the fused kernel also resets the id table for the next batch: keep that (two memsets)
    "no_agg": lambda: patch(sampler.MfgWorkspace, "aggregate", no_agg),
    "no_prep": lambda: (patch(sampler.MfgWorkspace, "run", lambda self, *a, **k: None),
                        patch(sampler.MfgWorkspace, "aggregate", lambda self, *a, **k: None)),
    "no_mbt": lambda: patch(model.FusedSAGE, "_input_grad", ig),
    "no_wgrad": lambda: patch(model.FusedSAGE, "_wgrad", lambda self, *a, **k: None),
}
for mode in sys.argv[1:] or list(modes):
    tr = Trainer(dg, train, TrainConfig(gather_free=True))
    tr.set_epoch(0)
    tr.begin_epoch(False)
    tr.run_steps(0, 4)
    torch.cuda.synchronize()
    modes[mode]()
    tr.graphs.clear()
    tr.run_steps(4, 4)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    tr.run_steps(8, 400)
    b.record()
    torch.cuda.synchronize()
    print(f"{mode:10s} {a.elapsed_time(b) / 400 * 1e3:7.1f} us/step", flush=True)
    unpatch()
