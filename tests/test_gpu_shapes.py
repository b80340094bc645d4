"""Drop-in parity at BASELINE.json's larger shapes (configs c2 arxiv, c3 products).

The graphs are generated on the device (synth_graph_device, the benchmark's
inputs); the oracle runs on host copies of the same arrays.  For batches of the
epoch plan (first, last, random) the public multihop_mfg digests at (15,10,5),
the paper order (5,10,15) and the inference fanout (20,20,20), and the
prepare_batch digests with f32 features (reference sampler.py:328-346,
prep.py:192-206), must equal the oracle's bit for bit.  The papers100M shape is
checked the same way by bench.py's parity gate (the `parity` key of its line).
"""
import numpy as np
import pytest

import oracle as O
import shape_parity as parity
from paper_2110_08450_b200 import make_epoch_plan
from paper_2110_08450_b200.graph import synth_graph_device

pytestmark = pytest.mark.gpu

SHAPES = {  # nodes, slots, features, classes, train ids
    "arxiv": (169_343, 1_166_243, 128, 40, 90_941),
    "products": (2_449_029, 61_859_140, 100, 47, 196_615),
}


@pytest.mark.parametrize("shape", list(SHAPES))
def test_shape_parity_against_oracle(shape):
    n, slots, f, c, ntrain = SHAPES[shape]
    dg = synth_graph_device(n, slots / n, 3.0, seed=1, num_features=f, num_classes=c,
                            feature_seed=1, label_seed=1)
    host = parity.host_copy(dg)
    train = np.sort(np.random.default_rng(1).choice(n, size=ntrain, replace=False))
    plan = make_epoch_plan(train, 1024, 1)
    batches = parity.pick_batches(plan, k=4, seed=3)
    r = parity.check(dg, host, batches, [(15, 10, 5), (5, 10, 15), (20, 20, 20)], 1)
    assert r["mismatches"] == [], r
    assert r["mfg_checked"] == 3 * len(batches) and r["batch_checked"] == len(batches)


def test_shape_parity_detects_a_wrong_graph():
    """The gate is not vacuous: one flipped neighbour id changes the digests."""
    n, slots, f, c, _ = SHAPES["arxiv"]
    dg = synth_graph_device(n, slots / n, 3.0, seed=1, num_features=f, num_classes=c)
    host = parity.host_copy(dg)
    plan = make_epoch_plan(np.arange(n), 1024, 1)
    b = plan.batches[0]
    # corrupt the host copy at a slot the first hop certainly reads: a seed whose
    # whole row is taken (0 < degree <= fanout)
    ip = host["indptr"]
    v = next(int(s) for s in b.dst_ids if 0 < ip[s + 1] - ip[s] <= 50)
    lo = int(ip[v])
    host["indices"] = host["indices"].copy()
    host["indices"][lo] = (host["indices"][lo] + 1) % n
    r = parity.check(dg, host, [b], [(50, 50)], 1, features=False)
    assert r["mfg_equal"] == 0 and len(r["mismatches"]) == 1
