"""f3 TRCE traces on the host: a trace written by the reference's record_trace
parses here, re-saves byte-identically, and malformed copies raise the
reference's errors (tests/golden/trace.npz)."""
import numpy as np
import pytest

from conftest import GOLDEN, golden
from paper_2110_08450_b200 import harness as S
from paper_2110_08450_b200 import files as F

TRACE = GOLDEN / "files" / "trace.trce"


def test_reference_trace_parses_and_roundtrips(tmp_path):
    z = golden("trace")
    tr = S.load_trace(TRACE)
    assert len(tr.records) == int(z["nrec"]) == 12
    assert tr.graph_checksum == int(z["checksum"]) and tr.global_seed == 11
    assert [r.hop for r in tr.records] == [0, 1, 2] * 4
    assert [r.fanout for r in tr.records] == [5, 10, 15] * 4
    assert [r.batch_id for r in tr.records[::3]] == z["batch_ids"].tolist()
    seeds = z["seeds"].reshape(4, 128)
    for b in range(4):
        assert np.array_equal(tr.records[3 * b].dst_ids, seeds[b])
    S.save_trace(tr, tmp_path / "t.trce")
    assert (tmp_path / "t.trce").read_bytes() == TRACE.read_bytes()
    assert tr.num_hops() == 3


def test_trace_errors_match_reference(tmp_path):
    z = golden("trace")
    good = TRACE.read_bytes()
    variants = {"badmagic": b"XXXX" + good[4:],
                "badversion": good[:4] + (2).to_bytes(4, "little") + good[8:],
                "trunc10": good[:10], "trunc40": good[:40], "trunc60": good[:60],
                "truncm1": good[:-1]}
    for tag, cls, msg in z["errors"]:
        p = tmp_path / tag
        p.write_bytes(variants[tag])
        with pytest.raises(getattr(F, cls)) as ei:
            S.load_trace(p)
        assert str(ei.value) == msg


def test_sweep_csv_and_grid():
    r = S.SweepResult(baseline="b", rows=[("b", 0, 0.001, 1.0), ("v", 0, 0.0005, 2.0)])
    assert r.to_csv() == ("variant,hop,time_s,speedup_vs_baseline\n"
                          "b,0,0.001000000,1.0000\nv,0,0.000500000,2.0000\n")
    descs = [v.descriptor for v in S.default_grid()]
    assert len(set(descs)) == len(descs) and S.DeviceVariant().descriptor in descs
