"""Run a few papers-shape training steps (target for `ncu -k regex:... --set full`).

ncu --set full -k regex:'sample_insert|mean_bwd_t' --launch-skip 30 -c 6 \
    -o gpurun_out/step python tools/ncu_step.py
"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2110_08450_b200.train import TrainConfig, Trainer  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
dg, train, _, _ = bench.build_data("papers")
tr = Trainer(dg, train, TrainConfig(gather_free=True))
tr.set_epoch(0)
tr.begin_epoch(False)
tr.run_steps(0, steps)
torch.cuda.synchronize()
print("done", tr.last_loss.item())
