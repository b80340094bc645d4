"""Standalone time of the two per-step chains (papers shape): prep (sample +
gather + transposes) alone, train (fwd + bwd + Adam) alone, and the overlapped
pair, each captured as a CUDA graph of R repetitions.

python tools/chains.py [key=val ...]   (TrainConfig overrides; under gpurun)
"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2110_08450_b200.train import TrainConfig, Trainer  # noqa: E402


def graph_time(fn, reps=20, iters=5):
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        fn()
        fn()
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / (reps * iters)


def main():
    kw = {}
    for a in sys.argv[1:]:
        k, v = a.split("=")
        f = TrainConfig.__dataclass_fields__[k]
        kw[k] = (v not in ("0", "false")) if f.type in (bool, "bool") else type(f.default)(v)
    dg, train, _, _ = bench.build_data("papers")
    tr = Trainer(dg, train, TrainConfig(gather_free=True, **kw))
    tr.set_epoch(0)
    tr.begin_epoch(False)
    tr.run_steps(0, 8)
    torch.cuda.synchronize()
    s0, s1 = tr.slots[:2]
    print(f"prep alone   {graph_time(lambda: tr._prep(s1, None, late=True)):7.1f} us")
    print(f"train alone  {graph_time(lambda: tr._train(s0)):7.1f} us")
    print(f"pair         {graph_time(lambda: tr._pair(0, False)):7.1f} us")


if __name__ == "__main__":
    main()
