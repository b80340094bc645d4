import os
import sys
from pathlib import Path

import numpy as np
import pytest

REPO = Path(__file__).resolve().parents[1]
GOLDEN = REPO / "tests" / "golden"
sys.path.insert(0, str(REPO))
sys.path.insert(0, str(REPO / "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running")


def golden(name):
    return np.load(GOLDEN / f"{name}.npz", allow_pickle=False)


@pytest.fixture(scope="session")
def g_small():
    return golden("graphs")


@pytest.fixture(scope="session")
def small_graph():
    from paper_2110_08450_b200 import synth_graph
    return synth_graph(1000, 8, 3.0, seed=13)


@pytest.fixture(scope="session")
def mfg_small():
    return golden("mfg_small")


@pytest.fixture(scope="session")
def prep_small():
    return golden("prep_small")


def gpu_available():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def golden_mfg(z, prefix):
    """(global_ids, layers) of one golden case, layers in consumption order."""
    gids = z[f"{prefix}global_ids"].astype(np.int64)
    layers = []
    i = 0
    while f"{prefix}l{i}_meta" in z:
        nd, ns, ne = (int(x) for x in z[f"{prefix}l{i}_meta"])
        layers.append(dict(num_dst=nd, num_src=ns, indptr=z[f"{prefix}l{i}_indptr"].astype(np.int64),
                           src_local=z[f"{prefix}l{i}_src"].astype(np.int64)))
        i += 1
    return gids, layers


def assert_mfg_equal(gids, layers, want_gids, want_layers):
    assert np.array_equal(np.asarray(gids, dtype=np.int64), want_gids)
    assert len(layers) == len(want_layers)
    for a, b in zip(layers, want_layers):
        assert (a["num_dst"], a["num_src"]) == (b["num_dst"], b["num_src"])
        assert np.array_equal(np.asarray(a["indptr"], dtype=np.int64), b["indptr"])
        assert np.array_equal(np.asarray(a["src_local"], dtype=np.int64), b["src_local"])
