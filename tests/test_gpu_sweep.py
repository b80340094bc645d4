"""f3 hop replay on the GPU: a trace recorded by the device sampler is
byte-identical to the one the reference recorded, and every device variant
replays it to the reference's own replay digest (bench.py:104-139)."""
import numpy as np
import pytest

from conftest import GOLDEN, golden
from paper_2110_08450_b200 import DeviceGraph, FanoutSpec, SeedBatch
from paper_2110_08450_b200.graph import CsrGraph
from paper_2110_08450_b200 import harness as S

pytestmark = pytest.mark.gpu
TRACE = GOLDEN / "files" / "trace.trce"


def _graph_and_plan():
    z = golden("trace")
    g = CsrGraph(5000, z["indptr"], z["indices"].astype(np.int64))
    seeds = z["seeds"].reshape(4, 128)

    class Plan:
        batches = [SeedBatch(int(b), seeds[i]) for i, b in enumerate(z["batch_ids"])]
    return z, DeviceGraph.from_host(g), Plan()


def test_record_trace_matches_reference_bytes(tmp_path):
    z, dg, plan = _graph_and_plan()
    assert S.graph_checksum(dg) == int(z["checksum"])
    S.record_trace(dg, plan, FanoutSpec((15, 10, 5)), 11, path=tmp_path / "t.trce")
    assert (tmp_path / "t.trce").read_bytes() == TRACE.read_bytes()


def test_every_variant_replays_to_reference_digest(tmp_path):
    z, dg, _ = _graph_and_plan()
    tr = S.load_trace(TRACE)
    want = str(z["digest"])
    assert S.replay_variant(tr, dg, S.DeviceVariant(), repetitions=1).digest == want
    res = S.sweep(tr, dg, S.default_grid(), S.DeviceVariant(), path=tmp_path / "s.csv",
                  repetitions=2)
    assert len(res.rows) == 3 * len(S.default_grid())
    assert (tmp_path / "s.csv").read_text().startswith("variant,hop,time_s")


def test_digest_mismatch_raises():
    z, dg, _ = _graph_and_plan()
    tr = S.load_trace(TRACE)
    bad = S.Trace(tr.graph_checksum, tr.global_seed + 1, tr.records)  # other draw streams
    a = S.replay_variant(bad, dg, S.DeviceVariant(), repetitions=1)
    assert a.digest != str(z["digest"])
    with pytest.raises(ValueError):
        S.replay_variant(S.Trace(123, 11, tr.records), dg, S.DeviceVariant())
