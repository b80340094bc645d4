"""GPU parity of slicing / prepare_batch / run_epoch_prep against reference goldens."""
import numpy as np
import pytest
import torch

import oracle as O
from conftest import golden
from paper_2110_08450_b200 import (DeviceGraph, FanoutSpec, FeatureMatrix, IdMap, LabelVector,
                                   PrepConfig, SamplerVariant, SeedBatch, from_edge_list,
                                   generate_features, generate_labels, make_epoch_plan,
                                   prepare_batch, run_epoch_prep, slice_features, slice_labels,
                                   synth_graph)
import paper_2110_08450_b200.prep as prep_mod

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def data13():
    g = synth_graph(1000, 8, 3.0, seed=13)
    return (g, DeviceGraph.from_host(g), generate_features(1000, 8, "f32", seed=13),
            generate_features(1000, 8, "f16", seed=13), generate_labels(1000, 7, seed=13))


def test_slice_features_identity_and_random(data13):
    _, _, fm32, fm16, _ = data13
    for fm in (fm32, fm16):
        idm = IdMap(SamplerVariant())
        idm.insert(np.arange(1000))
        out = torch.empty(1000 * 8, dtype=torch.float32, device="cuda")
        got = slice_features(fm, idm, out)
        assert got.cpu().numpy().tobytes() == fm.data.astype(np.float32).tobytes()
        ids = np.random.default_rng(2).choice(1000, size=100, replace=False)
        idm = IdMap(SamplerVariant())
        idm.insert(ids)
        got = slice_features(fm, idm, torch.empty(800, dtype=torch.float32, device="cuda"))
        assert np.array_equal(got.cpu().numpy(), O.gather_features(fm.data, ids))


def test_slice_features_f16_specials_bit_exact(prep_small):
    z = prep_small
    fm = FeatureMatrix(rows=4, cols=4, data=z["specials"].view(np.float16).reshape(4, 4))
    idm = IdMap(SamplerVariant())
    idm.insert(z["specials_ids"])
    got = slice_features(fm, idm, torch.empty(16, dtype=torch.float32, device="cuda"))
    assert np.array_equal(got.cpu().numpy().view(np.uint32), z["specials_out"])


def test_slice_features_capacity_error(data13):
    idm = IdMap(SamplerVariant())
    idm.insert(np.arange(10))
    with pytest.raises(ValueError, match="need"):
        slice_features(data13[2], idm, torch.empty(5, dtype=torch.float32, device="cuda"))


def test_slice_labels():
    y = LabelVector(values=np.array([9, 8, 7, 6]), num_classes=10)
    assert slice_labels(y, SeedBatch(0, np.array([3, 1]))).tolist() == [6, 8]
    assert len(slice_labels(y, SeedBatch(0, np.array([], dtype=np.int64)))) == 0


def test_prepare_batch_tiny_path():
    g = from_edge_list([(0, 1), (1, 2)], 3, make_undirected=True)
    fm = FeatureMatrix(rows=3, cols=1, data=np.array([[0.5], [1.5], [2.5]], dtype=np.float32))
    y = LabelVector(values=np.array([0, 1, 2]), num_classes=3)
    pb = prepare_batch(g, fm, y, SeedBatch(0, np.array([1])), FanoutSpec((2,)),
                       SamplerVariant(), 0)
    assert pb.mfg.id_map.global_ids.tolist() == [1, 0, 2]
    assert pb.features[:, 0].tolist() == [1.5, 0.5, 2.5]
    assert pb.labels.tolist() == [1]
    assert pb.byte_size > 0


def test_prepare_batch_isolated_seeds():
    g = from_edge_list([(3, 4)], 6)
    fm = generate_features(6, 2, "f32", seed=0)
    y = generate_labels(6, 2, seed=0)
    pb = prepare_batch(g, fm, y, SeedBatch(0, np.array([0, 1])), FanoutSpec((3, 3)),
                       SamplerVariant(), 0)
    assert pb.mfg.id_map.global_ids.tolist() == [0, 1]
    assert pb.mfg.num_edges == 0


def test_prepare_batch_digest_and_bytes_vs_reference(data13, prep_small):
    g, dg, _, fm16, y = data13
    z = prep_small
    plan = make_epoch_plan(np.arange(1000), 128, 5)
    pb = prepare_batch(dg, fm16, y, plan.batches[0], FanoutSpec((15, 10, 5)), SamplerVariant(),
                       42)
    assert np.array_equal(pb.features.cpu().numpy(), z["pb_features"])
    assert pb.labels.cpu().numpy().tolist() == z["pb_labels"].tolist()
    assert pb.digest() == str(z["pb_digest"])
    assert pb.byte_size == int(z["pb_byte_size"])
    assert pb.stats == tuple((l.num_dst, l.num_src, l.num_edges) for l in pb.mfg.layers)


def test_prepare_batch_sized_buffers_and_caller_slot(data13, prep_small):
    """prepare_batch sizes its feature rows to the MFG (reference _Slot.reserve), and a
    caller-kept slot gives the same batch; a slot built for other fanouts is refused."""
    g, dg, _, fm16, y = data13
    z = prep_small
    plan = make_epoch_plan(np.arange(1000), 128, 5)
    fan = FanoutSpec((15, 10, 5))
    pb = prepare_batch(dg, fm16, y, plan.batches[0], fan, SamplerVariant(), 42)
    assert pb.features.shape[0] == pb.num_nodes    # exact, not the worst-case capacity
    slot = prep_mod._Slot(dg, PrepConfig(fanouts=fan), 128, fm16.cols, dg.device)
    for _ in range(2):   # reusable
        pb2 = prepare_batch(dg, fm16, y, plan.batches[0], fan, SamplerVariant(), 42, slot=slot)
        assert pb2.digest() == str(z["pb_digest"])
    with pytest.raises(ValueError):
        prepare_batch(dg, fm16, y, plan.batches[0], FanoutSpec((3, 3)), SamplerVariant(), 42,
                      slot=slot)


@pytest.mark.parametrize("P", [2, 4])
def test_completion_order_delivery(data13, prep_small, P):
    """delivery='completion_order' (reference prep.py:289-305): every batch exactly once,
    each with the digest it has in plan order."""
    g, dg, fm32, fm16, y = data13
    z = prep_small
    plan = make_epoch_plan(np.arange(1000), 128, 5)
    run = run_epoch_prep(dg, fm16, y, plan, PrepConfig(num_workers=P, delivery="completion_order",
                                                       fanouts=FanoutSpec((15, 10, 5))), 42)
    got = {b.mfg.seeds.batch_id: b.digest() for b in run}
    assert sorted(got) == list(range(8))
    assert [got[i] for i in range(8)] == [str(d) for d in z["digests16"]]


@pytest.mark.parametrize("P", [1, 2, 4])
def test_epoch_digests_match_reference_any_depth(data13, prep_small, P):
    g, dg, fm32, fm16, y = data13
    z = prep_small
    plan = make_epoch_plan(np.arange(1000), 128, 5)
    for fm, key in ((fm32, "digests32"), (fm16, "digests16")):
        cfg = PrepConfig(num_workers=P, fanouts=FanoutSpec((15, 10, 5)))
        run = run_epoch_prep(dg, fm, y, plan, cfg, 42)
        got = [(b.mfg.seeds.batch_id, b.digest()) for b in run]
        assert [b for b, _ in got] == list(range(8))
        assert [d for _, d in got] == [str(d) for d in z[key]]
        # the reference's pool bound (prep.py:239): queue_capacity + num_workers buffers
        assert run.report.peak_resident <= min(cfg.depth + 1, P + cfg.queue_capacity)
        assert len(run.report.per_batch) == 8
        assert run.report.sampling_s > 0 and run.report.slicing_s > 0


def test_epoch_fp16_output_matches(data13):
    g, dg, _, fm16, y = data13
    plan = make_epoch_plan(np.arange(1000), 100, 3)
    a = [b.features.float().cpu().numpy() for b in run_epoch_prep(
        dg, fm16, y, plan, PrepConfig(fanouts=FanoutSpec((5, 5)), feature_dtype="f16"), 1)]
    b = [b.features.cpu().numpy() for b in run_epoch_prep(
        dg, fm16, y, plan, PrepConfig(fanouts=FanoutSpec((5, 5))), 1)]
    assert all(np.array_equal(x, y_) for x, y_ in zip(a, b))


def test_detach_survives_iteration(data13):
    g, dg, fm32, _, y = data13
    plan = make_epoch_plan(np.arange(1000), 256, 5)
    kept = []
    digests = []
    for b in run_epoch_prep(dg, fm32, y, plan, PrepConfig(num_workers=1,
                                                          fanouts=FanoutSpec((4, 4))), 7):
        digests.append(b.digest())
        kept.append(b.detach())
    assert [k.digest() for k in kept] == digests


def test_worker_error_propagates(data13, monkeypatch):
    g, dg, fm32, _, y = data13

    def boom(*a, **k):
        raise ValueError("sampling exploded")

    monkeypatch.setattr(prep_mod, "_prep_one", boom)
    plan = make_epoch_plan(np.arange(1000), 64, 5)
    with pytest.raises(RuntimeError, match="worker failed"):
        for _ in run_epoch_prep(dg, fm32, y, plan, PrepConfig(num_workers=2), 42):
            pass


def test_config1_prepared_batch_digests():
    """config 1 with 128-d f16 features and 172 classes: PreparedBatch digests."""
    z = golden("config1")
    g = synth_graph(100_000, 10, 3.0, seed=1)
    fm = generate_features(100_000, 128, "f16", seed=1)
    y = generate_labels(100_000, 172, seed=1)
    dg = DeviceGraph.from_host(g)
    plan = make_epoch_plan(np.arange(100_000), 1024, 1)
    want = {int(s[0]): str(d) for s, d in zip(z["stats"], z["batch_digests"])}
    got = {}
    for b in run_epoch_prep(dg, fm, y, plan, PrepConfig(num_workers=2), 1):
        if b.mfg.seeds.batch_id in want:
            got[b.mfg.seeds.batch_id] = b.digest()
    assert got == want
