"""f2 load throughput: the reference's MFGC/FEAT/LABL files -> one HBM replica.

Writes a products-shaped file set (2.45M nodes, ~62M slots, 100-d fp16,
47 classes) under $TMPDIR, then times (hot page cache, best of 3):
  ours      files.load_device_graph (pinned double-buffered streaming, device validation)
  host path the reference's loader restated (np.frombuffer + astype(int64) as in
            graph.py:203-249, CsrGraph.validate on the host) + DeviceGraph.from_host
python tools/load_bench.py [n_nodes] [avg_degree] [f]
"""
import json
import os
import sys
import tempfile
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2110_08450_b200 import files as F  # noqa: E402
from paper_2110_08450_b200.graph import (CsrGraph, DeviceGraph, FeatureMatrix,  # noqa: E402
                                         LabelVector, generate_labels)


def host_path(d):
    import struct
    with open(d / "g.mfgc", "rb") as f:
        f.read(8)
        n, e = struct.unpack("<QQ", f.read(16))
        indptr = np.frombuffer(f.read(8 * (n + 1)), dtype="<u8").astype(np.int64)
        indices = np.frombuffer(f.read(4 * e), dtype="<u4").astype(np.int64)
    g = CsrGraph(int(n), indptr, indices)
    g.validate()
    with open(d / "x.feat", "rb") as f:
        f.read(8)
        rows, cols, code = struct.unpack("<QIB3x", f.read(16))
        data = np.frombuffer(f.read(rows * cols * 2), dtype=np.float16).reshape(rows, cols)
    with open(d / "y.labl", "rb") as f:
        f.read(8)
        rows, nc = struct.unpack("<QI", f.read(12))
        vals = np.frombuffer(f.read(4 * rows), dtype="<u4").astype(np.int64)
    dg = DeviceGraph.from_host(g, FeatureMatrix(int(rows), int(cols), data),
                               LabelVector(vals, int(nc)))
    torch.cuda.synchronize()
    return dg


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 2_449_029
    deg = float(sys.argv[2]) if len(sys.argv) > 2 else 25.26
    f = int(sys.argv[3]) if len(sys.argv) > 3 else 100
    d = Path(tempfile.mkdtemp())
    t0 = time.perf_counter()
    # a device-generated graph of the synth_graph law, written with the reference format
    from paper_2110_08450_b200.graph import synth_graph_device
    src = synth_graph_device(n, deg, 3.0, seed=1, num_features=f, num_classes=47)
    g = CsrGraph(n, src.indptr.cpu().numpy(), src.indices.cpu().numpy())
    F.save_csr(g, d / "g.mfgc")
    F.save_features(FeatureMatrix(n, f, src.feature_view().cpu().numpy()), d / "x.feat")
    F.save_labels(LabelVector(src.labels.cpu().numpy(), 47), d / "y.labl")
    del src
    gen_s = time.perf_counter() - t0
    total = sum(os.path.getsize(d / x) for x in ("g.mfgc", "x.feat", "y.labl"))
    res = {}
    for name, fn in (("ours", lambda: F.load_device_graph(d / "g.mfgc", d / "x.feat",
                                                          d / "y.labl")),
                     ("host_path", lambda: host_path(d))):
        best = 1e9
        for _ in range(3):
            torch.cuda.synchronize()
            t = time.perf_counter()
            dg = fn()
            torch.cuda.synchronize()
            best = min(best, time.perf_counter() - t)
            del dg
            torch.cuda.empty_cache()
        res[name] = {"s": round(best, 4), "GBps": round(total / best / 1e9, 2)}
    a = F.load_device_graph(d / "g.mfgc", d / "x.feat", d / "y.labl")
    b = host_path(d)
    same = (torch.equal(a.indptr, b.indptr) and torch.equal(a.indices, b.indices)
            and torch.equal(a.feature_view(), b.feature_view()) and torch.equal(a.labels, b.labels))
    print(json.dumps({"files_bytes": total, "nodes": n, "edges": int(g.indptr[-1]), "f": f,
                      "write_s": round(gen_s, 1), "threads": F.READ_THREADS,
                      "identical": bool(same), **res}))


if __name__ == "__main__":
    main()
