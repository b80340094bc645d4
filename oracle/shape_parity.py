"""Parity of the device path against the CPU oracle on large shapes (TEST INFRASTRUCTURE ONLY).

Used by tests/test_gpu_shapes.py and by bench.py's parity gate (after its timed
region): for chosen batches of an epoch plan, the drop-in public API on the GPU
(multihop_mfg, prepare_batch) is compared digest for digest with the C oracle
(oracle.c, pinned to the reference's goldens by tests/test_oracle.py) run on
host copies of the SAME device-resident arrays.  Digests are the reference's
own: Mfg.digest (sampler.py:228-235) and PreparedBatch.digest (prep.py:132-137).
The oracle runs are spread over host threads (the ctypes calls release the GIL).
"""

from __future__ import annotations

import os
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

import oracle as O


def pick_batches(plan, k: int = 8, seed: int = 0):
    """First, last and k-2 seeded-random batches of the plan (plan order)."""
    nb = len(plan)
    if nb <= k:
        return list(plan.batches)
    rng = np.random.default_rng(seed)
    mid = rng.choice(np.arange(1, nb - 1), size=k - 2, replace=False)
    idx = sorted({0, nb - 1, *mid.tolist()})
    return [plan.batches[i] for i in idx]


def check(dg, host: dict, batches, fanout_sets, global_seed: int, features: bool = True,
          feature_fanouts=(15, 10, 5), nthreads: int | None = None) -> dict:
    """host: dict(indptr int64, indices int32, features [n, f] (fp16/f32) or None,
    labels int64 or None) — host copies of dg's arrays.

    Returns {"mfg_checked", "mfg_equal", "batch_checked", "batch_equal",
    "mismatches": [...], "seconds"}."""
    from paper_2110_08450_b200 import FanoutSpec, SamplerVariant, multihop_mfg, prepare_batch

    t0 = time.perf_counter()
    nthreads = nthreads or min(16, os.cpu_count() or 1)
    n = int(dg.num_nodes)
    ip, ind = host["indptr"], host["indices"]
    out = {"mfg_checked": 0, "mfg_equal": 0, "batch_checked": 0, "batch_equal": 0,
           "mismatches": []}

    def oracle_mfg(b, fan):
        gids, layers = O.multihop(ip, ind, n, b.dst_ids, fan, global_seed, b.batch_id)
        return gids, layers, O.mfg_digest(gids, layers)

    def oracle_batch(b, fan):
        gids, layers, hx = oracle_mfg(b, fan)
        feats = O.gather_features(host["features"], gids)
        labels = O.gather_labels(host["labels"], b.dst_ids)
        return O.batch_digest(hx, feats, labels)

    with ThreadPoolExecutor(nthreads) as pool:
        futs = {}
        for fan in fanout_sets:
            for b in batches:
                futs[("mfg", tuple(fan), b.batch_id)] = pool.submit(oracle_mfg, b, tuple(fan))
        if features and host.get("features") is not None:
            for b in batches:
                futs[("batch", tuple(feature_fanouts), b.batch_id)] = pool.submit(
                    oracle_batch, b, tuple(feature_fanouts))
        # device side meanwhile (one batch at a time through the public API)
        dev = {}
        for fan in fanout_sets:
            for b in batches:
                dev[("mfg", tuple(fan), b.batch_id)] = \
                    multihop_mfg(dg, b, FanoutSpec(tuple(fan)), global_seed).digest()
        if features and host.get("features") is not None:
            x = dg.feature_view()
            for b in batches:
                pb = prepare_batch(dg, x, dg.labels, b, FanoutSpec(tuple(feature_fanouts)),
                                   SamplerVariant(), global_seed)
                dev[("batch", tuple(feature_fanouts), b.batch_id)] = pb.digest()
                del pb
        for key, fut in futs.items():
            r = fut.result()
            want = r[2] if key[0] == "mfg" else r
            ok = dev[key] == want
            out[f"{key[0]}_checked"] += 1
            out[f"{key[0]}_equal"] += int(ok)
            if not ok:
                out["mismatches"].append({"kind": key[0], "fanouts": list(key[1]),
                                          "batch_id": int(key[2])})
    out["seconds"] = round(time.perf_counter() - t0, 2)
    return out


def host_copy(dg) -> dict:
    """Host copies of a DeviceGraph's arrays (features as the [n, f] view)."""
    x = dg.feature_view() if dg.features is not None else None
    return dict(indptr=dg.indptr.cpu().numpy(), indices=dg.indices.cpu().numpy(),
                features=None if x is None else np.ascontiguousarray(x.cpu().numpy()),
                labels=None if dg.labels is None else dg.labels.cpu().numpy())
