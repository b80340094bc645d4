"""The on-device generator (graph.synth_graph_device, csrc/generate.cu) against its
host restatement (oracle.synth_graph_host): bit-identical arrays, plus the law's
invariants at a size only the device builds quickly.  The law itself is checked
on the host arrays in tests/test_generate.py (reference graph.py:252-298)."""
import numpy as np
import pytest
import torch

import oracle as O
from paper_2110_08450_b200.graph import synth_graph_device

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,avg,f,c,seed", [(300_000, 14.55, 100, 47, 3),
                                            (50_001, 6.9, 128, 172, 1),
                                            (7, 3.0, 8, 2, 9)])
def test_device_generator_equals_host_restatement(n, avg, f, c, seed):
    dg = synth_graph_device(n, avg, 3.0, seed=seed, num_features=f, num_classes=c,
                            feature_seed=seed + 1, label_seed=seed + 2)
    torch.cuda.synchronize()
    h = O.synth_graph_host(n, avg, 3.0, seed=seed, num_features=f, num_classes=c,
                           feature_seed=seed + 1, label_seed=seed + 2, nthreads=8,
                           feature_stride=dg.features.shape[1])
    assert np.array_equal(dg.indptr.cpu().numpy(), h["indptr"])
    assert np.array_equal(dg.indices.cpu().numpy(), h["indices"])
    assert dg.features.cpu().numpy().view(np.uint16).tobytes() == \
        h["features"].view(np.uint16).tobytes()
    assert np.array_equal(dg.labels.cpu().numpy(), h["labels"])


def test_device_generator_invariants_large():
    """20M nodes (~290M slots): CSR valid, ids in range, even stub count, mean
    degree, and the directed slot multiset equal to its transpose (every pair
    stored in both directions) — checked on the device by sorting."""
    n, avg = 20_000_000, 14.55
    dg = synth_graph_device(n, avg, 3.0, seed=21)
    ip, ind = dg.indptr, dg.indices
    E = int(ip[-1].item())
    assert int(ip[0].item()) == 0 and E == ind.numel() and E % 2 == 0
    assert bool((ip[1:] >= ip[:-1]).all())
    assert int(ind.min().item()) >= 0 and int(ind.max().item()) < n
    assert abs(E / n - avg) / avg < 0.02
    owner = torch.repeat_interleave(torch.arange(n, device="cuda", dtype=torch.int64),
                                    (ip[1:] - ip[:-1]))
    i64 = ind.to(torch.int64)
    fwd = torch.sort(owner * n + i64).values
    rev = torch.sort(i64 * n + owner).values
    assert torch.equal(fwd, rev)
