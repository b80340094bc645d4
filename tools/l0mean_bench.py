"""Layer-0 mean (gather-free, rows from the HBM table) timed alone on papers-shape
batches: B batches sampled once, then the mean kernel replayed in a CUDA graph.

python tools/l0mean_bench.py [batches] [reps]   
"""
import json
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2110_08450_b200 import _lib  # noqa: E402
from paper_2110_08450_b200.sampler import MfgWorkspace  # noqa: E402
from paper_2110_08450_b200.train import TrainConfig, Trainer  # noqa: E402


def main():
    nb = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    dg, train, _, _ = bench.build_data("papers")
    tr = Trainer(dg, train, TrainConfig(gather_free=True, graphs=False))
    tr.set_epoch(0)
    L = _lib.lib()
    x = tr.x_table
    f = x.shape[1]
    wss, outs = [], []
    e0 = 0
    for b in range(nb):
        ws = MfgWorkspace(dg.num_nodes, tr.cfg.fanouts, 1024, last_hop_edges=True)
        ws.run(dg, tr.seeds_all, tr.desc_all[b], 1, tr.policy)
        wss.append(ws)
        outs.append(torch.empty((ws.node_cap[2], f), dtype=torch.bfloat16, device="cuda"))
    torch.cuda.synchronize()
    d0 = 0
    for ws in wss:
        s, e = ws.read_extents()
        e0 += e[2]
        d0 += s[2]

    def run():
        for ws, o in zip(wss, outs):
            _lib.check(L.sal_segment_mean_fwd(
                ws.dst_indptr[2].data_ptr(), ws.src_glob.data_ptr(), ws.sizes[2:3].data_ptr(),
                ws.node_cap[2], x.data_ptr(), _lib.SAL_F16, x.stride(0), f, o.data_ptr(),
                _lib.SAL_BF16, o.stride(0), _lib.stream_ptr()), "mean")
    run()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        run()
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(reps):
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) / nb)
    byts = (e0 * (f * 2 + 4) + d0 * (4 + f * 2)) / nb
    print(json.dumps({"us": round(best * 1e3, 2),
                      "GBps": round(byts / best / 1e6, 1), "edges": e0 / nb}))


if __name__ == "__main__":
    main()
